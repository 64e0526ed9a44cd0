// kernels.cu -- the CUDA kernels of the IGS-GMRES hot path for B200 (sm_100a).
//
// P:n = PAPER.md line n (arXiv 2205.07805).  Every kernel is FP64 and HBM- or
// latency-bound: no tensor cores on the iteration path.
//
//   spmv_kernel          z = A u, CSR, LPR lanes per row            (Alg. 3 Step 4)
//   bdot_kernel          [V_p, u]^T [u, z], one read of V_p, deterministic two-stage
//                        reduction, last CTA finishes
//   small_kernel         one CTA: (I+L)^{-1} r2, lagged norm, Stephen's trick, H column,
//                        Givens, status
//   update_kernel        v_p = (u - V_p r2)/gamma, u' = z/gamma - V_{p+1} r1, one read of
//                        V_p (the paper's "merge ... into one GPU kernel")
//   xupdate_kernel       x += V_p y
//   gram/loo kernels     ||I - V^T V||_F diagnostic
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "igs_internal.cuh"
#include "ptx_util.cuh"
#include "xchg.cuh"

namespace igs {

#define FULL_MASK 0xffffffffu

// ------------------------------------------------------------------------------------
// small utilities
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double2 ld2_guard(const double* __restrict__ p, int64_t r, int64_t n) {
    if (r + 1 < n) return __ldg(reinterpret_cast<const double2*>(p + r));
    double2 v;
    v.x = (r < n) ? __ldg(p + r) : 0.0;
    v.y = 0.0;
    return v;
}

__device__ __forceinline__ bool running(const int* istate) {
    return istate == nullptr || *(volatile const int*)(istate + ST_STATUS) == RUNNING;
}

// ------------------------------------------------------------------------------------
// K1: CSR SpMV with LPR lanes per row (LPR in {1,2,4,8,16,32}).
//   Local column space: c < nloc -> x[c], else ghost[c - nloc] (halo, multi-GPU).
// ------------------------------------------------------------------------------------
template <int LPR, typename IT, typename PT, bool GHOST, bool RESID>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t nrows, const PT* __restrict__ rowptr,
                                                   const IT* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ ghost, int64_t nloc,
                                                   double* __restrict__ y,
                                                   const double* __restrict__ b,
                                                   const int* istate) {
    if (!running(istate)) return;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = gtid / LPR;
    const int sub = threadIdx.x % LPR;
    const bool valid = row < nrows;  // no early exit: the whole warp joins the shuffles
    const int64_t q0 = valid ? (int64_t)__ldg(rowptr + row) : 0;
    const int64_t q1 = valid ? (int64_t)__ldg(rowptr + row + 1) : 0;
    double s = 0.0;
    for (int64_t q = q0 + sub; q < q1; q += LPR) {
        const int64_t c = (int64_t)__ldg(col + q);
        double xv;
        if (GHOST && c >= nloc) xv = __ldg(ghost + (c - nloc));
        else xv = __ldg(x + c);
        s = fma(__ldg(val + q), xv, s);
    }
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) s += __shfl_xor_sync(FULL_MASK, s, off, LPR);
    if (valid && sub == 0) y[row] = RESID ? b[row] - s : s;
}

// CSR-stream SpMV for short rows (mean <= SPS_MAX_AVG nnz/row): a CTA owns 256 consecutive
// rows; its products val[q]*x[col[q]] are formed with fully coalesced val/col loads into
// shared memory, then thread t sums row t's products left to right -- the same rounding
// sequence as a sequential CSR row loop (product, then add), with none of the per-row
// lane waste of vector CSR at ~7 nnz/row.
constexpr int SPS_THREADS = 256;
constexpr int SPS_ROWS = 256;                // rows per CTA for R = 1 (R rows per thread)
constexpr int SPS_K = 8;                     // staged nonzeros per thread per row of R

template <int R, typename IT, typename PT, bool GHOST, bool RESID>
__global__ void __launch_bounds__(SPS_THREADS)
    spmv_stream_kernel(int64_t nrows, const PT* __restrict__ rowptr, const IT* __restrict__ col,
                       const double* __restrict__ val, const double* __restrict__ x,
                       const double* __restrict__ ghost, int64_t nloc, double* __restrict__ y,
                       const double* __restrict__ b, const int* istate) {
    if (!running(istate)) return;
    constexpr int ROWS = SPS_ROWS * R, K = SPS_K * R, CAP = ROWS * SPS_K;
    __shared__ double prod[CAP];
    const int64_t r0 = (int64_t)blockIdx.x * ROWS;
    const int64_t rl = (r0 + ROWS < nrows) ? r0 + ROWS : nrows;
    const int64_t q0 = (int64_t)__ldg(rowptr + r0), q1 = (int64_t)__ldg(rowptr + rl);
    const int cnt = (int)(q1 - q0 < (int64_t)CAP + 1 ? q1 - q0 : (int64_t)CAP + 1);
    int ra[R], re[R];
#pragma unroll
    for (int j = 0; j < R; j++) {
        const int64_t r = r0 + threadIdx.x + j * SPS_THREADS;
        ra[j] = re[j] = 0;
        if (r < nrows) { ra[j] = (int)((int64_t)__ldg(rowptr + r) - q0); re[j] = (int)((int64_t)__ldg(rowptr + r + 1) - q0); }
    }
    if (cnt <= CAP) {
        // all column and value loads first, then all gathers: 3 x K independent loads per thread
        int64_t cc[K];
        double vv[K], xv[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int i = threadIdx.x + k * SPS_THREADS;
            cc[k] = i < cnt ? (int64_t)__ldg(col + q0 + i) : 0;
            vv[k] = i < cnt ? __ldg(val + q0 + i) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int i = threadIdx.x + k * SPS_THREADS;
            if (GHOST && cc[k] >= nloc) xv[k] = i < cnt ? __ldg(ghost + (cc[k] - nloc)) : 0.0;
            else xv[k] = i < cnt ? __ldg(x + cc[k]) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int i = threadIdx.x + k * SPS_THREADS;
            if (i < cnt) prod[i] = __dmul_rn(vv[k], xv[k]);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int64_t r = r0 + threadIdx.x + j * SPS_THREADS;
            if (r < nrows) {
                double sum = 0.0;
                for (int q = ra[j]; q < re[j]; q++) sum = __dadd_rn(sum, prod[q]);
                y[r] = RESID ? b[r] - sum : sum;
            }
        }
    } else {  // more than SPS_K nonzeros per row on average here: row loop
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int64_t r = r0 + threadIdx.x + j * SPS_THREADS;
            if (r >= nrows) continue;
            double sum = 0.0;
            for (int64_t q = q0 + ra[j]; q < q0 + re[j]; q++) {
                const int64_t c = (int64_t)__ldg(col + q);
                const double xq = (GHOST && c >= nloc) ? __ldg(ghost + (c - nloc)) : __ldg(x + c);
                sum = __dadd_rn(sum, __dmul_rn(__ldg(val + q), xq));
            }
            y[r] = RESID ? b[r] - sum : sum;
        }
    }
}

// ------------------------------------------------------------------------------------
// K1 (default for short rows): the SELL-32 copy of A, with diagonal slices
// ------------------------------------------------------------------------------------
constexpr int SELL_THREADS = 256;

// The SELL-32 arrays as the kernels see them (SpmvArgs, igs_internal.cuh).
template <typename IT>
struct SellDev {
    const int64_t* __restrict__ ptr;   // [nslices + 1] value offset of slice s
    const int64_t* __restrict__ cptr;  // [nslices + 1] column offset; cptr[s+1] == cptr[s]: diagonal
    const int32_t* __restrict__ diag;  // [nslices * 8] offsets of a diagonal slice, ascending
    const uint8_t* __restrict__ len;   // [nrows]
    const uint8_t* __restrict__ mask;  // [nrows] offsets a row of a diagonal slice uses
    const IT* __restrict__ col;
    const double* __restrict__ val;
};

template <typename IT>
static SellDev<IT> sell_dev(const SpmvArgs& a) {
    return SellDev<IT>{a.sell_ptr, a.sell_cptr, a.sell_diag, a.sell_len, a.sell_mask,
                       static_cast<const IT*>(a.sell_col), a.sell_val};
}

template <bool CG>
__device__ __forceinline__ double ldx(const double* p) {
    if (CG) return __ldcg(p);  // written earlier in the same launch (persistent kernel)
    return __ldg(p);
}

// Row r of the SELL-32 copy, summed left to right in the row's CSR order with separate
// multiply and add (bitwise the oracle's row loop).  Called by all 32 lanes of a warp for
// the 32 rows of slice r >> 5 (rows >= nrows pass valid = false).  In a diagonal slice the
// column of an entry is r + offset, the offset one of the slice's list (read by every lane:
// one 32-byte broadcast) and the entries present named by the row's mask (no column index is
// read: 4 or 8 bytes less per nonzero, and the x gathers no longer wait for a column
// load).  Returns false for rows it must not store (past the end, boundary).
// KIND: SELL_MIXED (either slice kind), SELL_ALL_DIAG (every slice diagonal: no column
// offsets read, no explicit path compiled -- fewer registers, more resident warps),
// SELL_NO_DIAG (every slice explicit).
enum { SELL_MIXED = 0, SELL_ALL_DIAG = 1, SELL_NO_DIAG = 2 };

template <typename IT, bool GHOST, bool CG, int KIND>
__device__ __forceinline__ bool sell_row(const SellDev<IT>& A, int64_t r, bool valid, const double* __restrict__ x,
                                         const double* __restrict__ ghost, int64_t nloc, double& out) {
    const int64_t s = r >> 5;
    int len = valid ? (int)__ldg(A.len + r) : 0;
    const bool bnd = (len == SELL_BOUNDARY);  // G > 1 boundary row: launch_spmv_rows, after the halo
    if (bnd) len = 0;
    const int64_t base = __ldg(A.ptr + s) + (r & 31);
    int64_t cb = 0, ce = 0;
    if (KIND == SELL_MIXED) { cb = __ldg(A.cptr + s); ce = __ldg(A.cptr + s + 1); }
    if (KIND == SELL_NO_DIAG) cb = __ldg(A.cptr + s);
    double sum = 0.0;
    if (KIND == SELL_ALL_DIAG || (KIND == SELL_MIXED && ce == cb)) {  // diagonal (or empty) slice: warp-uniform
        // stored by list position: the entry with offset list[j] of row 32s+l at ptr[s] + 32j + l,
        // present iff bit j of the row's mask; the list ascends like the row's columns, so
        // position order is the row's CSR order.  Value loads: one base + immediates; nothing
        // depends on the row length (it only marks boundary rows, which have mask 0).
        const int4 d0 = __ldg(reinterpret_cast<const int4*>(A.diag + 8 * s));
        const int4 d1 = __ldg(reinterpret_cast<const int4*>(A.diag + 8 * s) + 1);
        const int dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        const unsigned m = valid ? (unsigned)__ldg(A.mask + r) : 0u;
        const char* xb = reinterpret_cast<const char*>(x + r);
        const double* vp = A.val + base;
        // Absent positions contribute 0.0 * 0.0 = +0.0 (neither the padding nor x is read):
        // a sum that starts at +0.0 is never -0.0, so adding +0.0 leaves every bit of it --
        // the 8 multiply-adds run unconditionally and equal the row's own shorter sum.
        double vv[8], xv[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            vv[j] = 0.0;
            xv[j] = 0.0;
            if ((m >> j) & 1u) {
                vv[j] = __ldg(vp + 32 * j);
                xv[j] = ldx<CG>(reinterpret_cast<const double*>(xb + 8 * (int64_t)dd[j]));
            }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) sum = __dadd_rn(sum, __dmul_rn(vv[j], xv[j]));
    } else if (KIND != SELL_ALL_DIAG) {
        const int64_t cbase = cb + (r & 31);
        for (int k0 = 0; k0 < len; k0 += 8) {
            IT cc[8];
            double vv[8], xv[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const bool in = k0 + k < len;
                cc[k] = in ? __ldg(A.col + cbase + 32 * (int64_t)(k0 + k)) : (IT)0;
                vv[k] = in ? __ldg(A.val + base + 32 * (int64_t)(k0 + k)) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (k0 + k < len) {
                    if (GHOST && (int64_t)cc[k] >= nloc) xv[k] = __ldg(ghost + ((int64_t)cc[k] - nloc));
                    else xv[k] = ldx<CG>(x + (int64_t)cc[k]);
                } else {
                    xv[k] = 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (k0 + k < len) sum = __dadd_rn(sum, __dmul_rn(vv[k], xv[k]));
        }
    }
    out = sum;
    return valid && !bnd;
}

// K1 (default for short rows): SELL-32.  One thread per row; the k-th nonzero of the 32
// rows of a slice are 32 consecutive entries, so the value (and column) loads of a warp
// are fully coalesced and, for stencil rows, the x gathers of a warp are one contiguous
// range per k.  No shared memory, no barrier.  8 entries per batch are loaded before use
// (memory-level parallelism).
template <typename IT, bool GHOST, bool RESID, int KIND>
__global__ void __launch_bounds__(SELL_THREADS, KIND == SELL_ALL_DIAG ? 5 : 1)
    spmv_sell_kernel(int64_t nrows, SellDev<IT> A, const double* __restrict__ x, const double* __restrict__ ghost,
                     int64_t nloc, double* __restrict__ y, const double* __restrict__ b, const int* istate,
                     int ahead) {
    // the status word gates only the store: its load overlaps the row's first loads (a
    // stopped solve's SpMV computes and discards; x is always a valid vector)
    const bool live = running(istate);
    if (ahead > 0 && threadIdx.x == 0 && live) {
        // the CTA that runs about one resident wave later: its values (and columns) to L2 now
        const int64_t nb = (int64_t)gridDim.x, fb = (int64_t)blockIdx.x + ahead;
        if (fb < nb) {
            const int64_t ns = (nrows + 31) / 32;
            const int64_t s0 = fb * (SELL_THREADS / 32), s1 = min(s0 + SELL_THREADS / 32, ns);
            const int64_t e0 = __ldg(A.ptr + s0), e1 = __ldg(A.ptr + s1);
            if (e1 > e0) bulk_prefetch_l2(A.val + e0, (uint32_t)((e1 - e0) * sizeof(double)));
            if (KIND != SELL_ALL_DIAG) {  // column indices of its explicit slices (contiguous)
                const int64_t c0 = __ldg(A.cptr + s0), c1 = __ldg(A.cptr + s1);
                if (c1 > c0) bulk_prefetch_l2(A.col + c0, (uint32_t)((c1 - c0) * sizeof(IT)));
            }
            // and the row lengths / masks / slice offsets its first loads wait on
            const int64_t r0 = s0 * 32, nr = min(s1 * 32, nrows) - r0;
            bulk_prefetch_l2(A.len + (r0 & ~(int64_t)15), (uint32_t)((nr + 31) & ~31));
            if (KIND != SELL_NO_DIAG) {
                bulk_prefetch_l2(A.mask + (r0 & ~(int64_t)15), (uint32_t)((nr + 31) & ~31));
                bulk_prefetch_l2(A.diag + 8 * s0, (uint32_t)(32 * (s1 - s0)));
            }
        }
    }
    const int64_t r = (int64_t)blockIdx.x * SELL_THREADS + threadIdx.x;
    if ((r & ~(int64_t)31) >= nrows) return;  // whole warps only (sell_row shuffles)
    double sum;
    const bool st = sell_row<IT, GHOST, false, KIND>(A, r, r < nrows, x, ghost, nloc, sum);
    if (st && live) y[r] = RESID ? b[r] - sum : sum;
}

// K1 for matrices whose slices are all diagonal (the stencil configs c1, c3, c4, c5): resident
// CTAs, each warp walking slices s, s + W, s + 2W, ... (W = warps in the grid), software-
// pipelined by one slice.  A slice costs two dependent rounds of loads: its metadata (value
// offset, masks, boundary marks, offset list: ~100 bytes per warp) and then its values and x
// gathers (~2 KB per warp).  With one short-lived warp per slice half of the resident warps
// sit in the first round, where they keep almost nothing in flight (ncu: 31 warps per SM,
// 5.9 TB/s, issue slots 30% busy, every stall a long-scoreboard wait); here the metadata of
// slice s + W is requested before the values of slice s, so every resident warp always has
// a slice's values and gathers in flight.  Same arithmetic as sell_row.
constexpr int SD_CTAS_PER_SM = 4;

template <bool RESID>
__global__ void __launch_bounds__(SELL_THREADS, SD_CTAS_PER_SM)
    spmv_sell_diag_kernel(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ diag,
                          const uint8_t* __restrict__ len8, const uint8_t* __restrict__ mask8,
                          const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                          const double* __restrict__ b, const int* istate) {
    if (!running(istate)) return;
    const int lane = threadIdx.x & 31;
    const int64_t ns = (nrows + 31) >> 5;
    const int64_t W = (int64_t)gridDim.x * (SELL_THREADS / 32);
    int64_t s = (int64_t)blockIdx.x * (SELL_THREADS / 32) + (threadIdx.x >> 5);
    if (s >= ns) return;
    // round 1 of the first slice (masks / lengths are padded to whole slices)
    int64_t p0 = __ldg(ptr + s);
    unsigned m = __ldg(mask8 + 32 * s + lane), ln = __ldg(len8 + 32 * s + lane);
    int4 d0 = __ldg(reinterpret_cast<const int4*>(diag + 8 * s));
    int4 d1 = __ldg(reinterpret_cast<const int4*>(diag + 8 * s) + 1);
    for (;;) {
        const int64_t sn = s + W;
        const bool more = sn < ns;  // warp-uniform
        int64_t p0n = 0;
        unsigned mn = 0, lnn = 0;
        int4 d0n = make_int4(0, 0, 0, 0), d1n = d0n;
        if (more) {  // round 1 of the next slice, in flight during round 2 of this one
            p0n = __ldg(ptr + sn);
            mn = __ldg(mask8 + 32 * sn + lane);
            lnn = __ldg(len8 + 32 * sn + lane);
            d0n = __ldg(reinterpret_cast<const int4*>(diag + 8 * sn));
            d1n = __ldg(reinterpret_cast<const int4*>(diag + 8 * sn) + 1);
        }
        const int64_t r = 32 * s + lane;
        const char* xb = reinterpret_cast<const char*>(x + r);
        const double* vp = val + p0 + lane;
        const int dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        double vv[8], xv[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            vv[j] = 0.0;
            xv[j] = 0.0;
            if ((m >> j) & 1u) {
                vv[j] = __ldg(vp + 32 * j);
                xv[j] = __ldg(reinterpret_cast<const double*>(xb + 8 * (int64_t)dd[j]));
            }
        }
        const bool st = r < nrows && ln != SELL_BOUNDARY;  // boundary rows (G > 1): launch_spmv_rows
        double bv = 0.0;
        if (RESID && st) bv = __ldg(b + r);
        double sum = 0.0;  // absent positions add 0.0 * 0.0 = +0.0: no bit of the sum changes (sell_row)
#pragma unroll
        for (int j = 0; j < 8; j++) sum = __dadd_rn(sum, __dmul_rn(vv[j], xv[j]));
        if (st) y[r] = RESID ? bv - sum : sum;
        if (!more) break;
        s = sn; p0 = p0n; m = mn; ln = lnn; d0 = d0n; d1 = d1n;
    }
}

static void spmv_sell_diag(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                           const int* istate, cudaStream_t s) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t blocks = (a.nrows + SELL_THREADS - 1) / SELL_THREADS;
    const unsigned grid = (unsigned)std::min<int64_t>(blocks, (int64_t)SD_CTAS_PER_SM * sms);
    if (resid) spmv_sell_diag_kernel<true><<<grid, SELL_THREADS, 0, s>>>(a.nrows, a.sell_ptr, a.sell_diag, a.sell_len, a.sell_mask, a.sell_val, x, y, b, istate);
    else spmv_sell_diag_kernel<false><<<grid, SELL_THREADS, 0, s>>>(a.nrows, a.sell_ptr, a.sell_diag, a.sell_len, a.sell_mask, a.sell_val, x, y, b, istate);
}

template <typename IT>
static void spmv_sell(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                      const int* istate, cudaStream_t s) {
    const unsigned blocks = (unsigned)((a.nrows + SELL_THREADS - 1) / SELL_THREADS);
    if (blocks == 0) return;
    if (a.sell_kind == SELL_ALL_DIAG && a.sell_walk_min_n >= 0 && a.nrows >= a.sell_walk_min_n) {
        spmv_sell_diag(a, x, y, b, resid, istate, s);
        return;
    }
    // L2 prefetch distance in CTAs: about one resident wave (4 CTAs per SM of 256 threads).
    // c4: 5.5 -> 6.4 TB/s (the latency of the dependent value/column -> gather phases now
    // hits L2 instead of DRAM)
    static int ahead = -1;
    if (ahead < 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        ahead = 4 * sms;
    }
    const SellDev<IT> A = sell_dev<IT>(a);
    const double* g = a.ghost;
    switch (a.sell_kind * 4 + (g ? 2 : 0) + (resid ? 1 : 0)) {
#define IGS_SELL_CASE(K, GH, RS)                                                                            \
    case K * 4 + (GH ? 2 : 0) + (RS ? 1 : 0):                                                             \
        spmv_sell_kernel<IT, GH, RS, K><<<blocks, SELL_THREADS, 0, s>>>(a.nrows, A, x, g, a.nloc, y, b, istate, ahead); \
        break;
        IGS_SELL_CASE(SELL_MIXED, false, false) IGS_SELL_CASE(SELL_MIXED, false, true)
        IGS_SELL_CASE(SELL_MIXED, true, false) IGS_SELL_CASE(SELL_MIXED, true, true)
        IGS_SELL_CASE(SELL_ALL_DIAG, false, false) IGS_SELL_CASE(SELL_ALL_DIAG, false, true)
        IGS_SELL_CASE(SELL_ALL_DIAG, true, false) IGS_SELL_CASE(SELL_ALL_DIAG, true, true)
        IGS_SELL_CASE(SELL_NO_DIAG, false, false) IGS_SELL_CASE(SELL_NO_DIAG, false, true)
        IGS_SELL_CASE(SELL_NO_DIAG, true, false) IGS_SELL_CASE(SELL_NO_DIAG, true, true)
#undef IGS_SELL_CASE
        default: break;
    }
}

// Boundary rows (G > 1): one thread per listed row rows[t], whose entries are entries
// rowptr[t]..rowptr[t+1] of the compact boundary-row CSR (igs_create keeps only these rows
// next to the SELL copy), ghosts for columns >= nloc, separate multiply and add left to
// right (the same rounding as the SELL / CSR kernels).
template <typename IT, typename PT, bool RESID>
__global__ void __launch_bounds__(256)
    spmv_rows_kernel(int64_t nb, const int64_t* __restrict__ rows, const PT* __restrict__ rowptr,
                     const IT* __restrict__ col, const double* __restrict__ val,
                     const double* __restrict__ x, const double* __restrict__ ghost, int64_t nloc,
                     double* __restrict__ y, const double* __restrict__ b, const int* istate) {
    if (!running(istate)) return;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nb) return;
    const int64_t r = __ldg(rows + t);
    double sum = 0.0;
    const int64_t q1 = (int64_t)__ldg(rowptr + t + 1);
    for (int64_t q = (int64_t)__ldg(rowptr + t); q < q1; q++) {
        const int64_t c = (int64_t)__ldg(col + q);
        const double xv = c >= nloc ? __ldg(ghost + (c - nloc)) : __ldg(x + c);
        sum = __dadd_rn(sum, __dmul_rn(__ldg(val + q), xv));
    }
    y[r] = RESID ? b[r] - sum : sum;
}

template <typename IT, typename PT>
static void spmv_rows_t(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                        const int* istate, cudaStream_t s) {
    const unsigned blocks = (unsigned)((a.n_bnd + 255) / 256);
    if (blocks == 0) return;
    const PT* rp = static_cast<const PT*>(a.rowptr);
    const IT* ci = static_cast<const IT*>(a.col);
    if (resid) spmv_rows_kernel<IT, PT, true><<<blocks, 256, 0, s>>>(a.n_bnd, a.bnd_rows, rp, ci, a.val, x, a.ghost, a.nloc, y, b, istate);
    else spmv_rows_kernel<IT, PT, false><<<blocks, 256, 0, s>>>(a.n_bnd, a.bnd_rows, rp, ci, a.val, x, a.ghost, a.nloc, y, b, istate);
}

void launch_spmv_rows(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                      const int* istate, cudaStream_t s) {
    if (a.idx64) {
        if (a.ptr64) spmv_rows_t<int64_t, int64_t>(a, x, y, b, resid, istate, s);
        else spmv_rows_t<int64_t, int32_t>(a, x, y, b, resid, istate, s);
    } else {
        if (a.ptr64) spmv_rows_t<int32_t, int64_t>(a, x, y, b, resid, istate, s);
        else spmv_rows_t<int32_t, int32_t>(a, x, y, b, resid, istate, s);
    }
}

template <typename IT, typename PT>
static void spmv_stream(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                        const int* istate, cudaStream_t s) {
    constexpr int R = 1;  // rows per thread
    const unsigned blocks = (unsigned)((a.nrows + SPS_ROWS * R - 1) / (SPS_ROWS * R));
    if (blocks == 0) return;
    const PT* rp = static_cast<const PT*>(a.rowptr);
    const IT* ci = static_cast<const IT*>(a.col);
    if (a.ghost) {
        if (resid) spmv_stream_kernel<R, IT, PT, true, true><<<blocks, SPS_THREADS, 0, s>>>(a.nrows, rp, ci, a.val, x, a.ghost, a.nloc, y, b, istate);
        else spmv_stream_kernel<R, IT, PT, true, false><<<blocks, SPS_THREADS, 0, s>>>(a.nrows, rp, ci, a.val, x, a.ghost, a.nloc, y, b, istate);
    } else {
        if (resid) spmv_stream_kernel<R, IT, PT, false, true><<<blocks, SPS_THREADS, 0, s>>>(a.nrows, rp, ci, a.val, x, nullptr, a.nloc, y, b, istate);
        else spmv_stream_kernel<R, IT, PT, false, false><<<blocks, SPS_THREADS, 0, s>>>(a.nrows, rp, ci, a.val, x, nullptr, a.nloc, y, b, istate);
    }
}

template <int LPR, typename IT, typename PT>
static void spmv_dispatch_g(const SpmvArgs& a, const double* x, double* y, const double* b,
                            bool resid, const int* istate, cudaStream_t s) {
    const int threads = 256;
    const int64_t nthreads = a.nrows * LPR;
    const unsigned blocks = (unsigned)((nthreads + threads - 1) / threads);
    if (blocks == 0) return;
    const PT* rp = static_cast<const PT*>(a.rowptr);
    const IT* ci = static_cast<const IT*>(a.col);
    if (a.ghost) {
        if (resid) spmv_kernel<LPR, IT, PT, true, true><<<blocks, threads, 0, s>>>(a.nrows, rp, ci, a.val, x, a.ghost, a.nloc, y, b, istate);
        else spmv_kernel<LPR, IT, PT, true, false><<<blocks, threads, 0, s>>>(a.nrows, rp, ci, a.val, x, a.ghost, a.nloc, y, b, istate);
    } else {
        if (resid) spmv_kernel<LPR, IT, PT, false, true><<<blocks, threads, 0, s>>>(a.nrows, rp, ci, a.val, x, nullptr, a.nloc, y, b, istate);
        else spmv_kernel<LPR, IT, PT, false, false><<<blocks, threads, 0, s>>>(a.nrows, rp, ci, a.val, x, nullptr, a.nloc, y, b, istate);
    }
}

template <typename IT, typename PT>
static void spmv_dispatch_l(const SpmvArgs& a, const double* x, double* y, const double* b,
                            bool resid, const int* istate, cudaStream_t s) {
    if (a.lpr == 0) { spmv_stream<IT, PT>(a, x, y, b, resid, istate, s); return; }
    switch (a.lpr) {
        case 1: spmv_dispatch_g<1, IT, PT>(a, x, y, b, resid, istate, s); break;
        case 2: spmv_dispatch_g<2, IT, PT>(a, x, y, b, resid, istate, s); break;
        case 4: spmv_dispatch_g<4, IT, PT>(a, x, y, b, resid, istate, s); break;
        case 8: spmv_dispatch_g<8, IT, PT>(a, x, y, b, resid, istate, s); break;
        case 16: spmv_dispatch_g<16, IT, PT>(a, x, y, b, resid, istate, s); break;
        default: spmv_dispatch_g<32, IT, PT>(a, x, y, b, resid, istate, s); break;
    }
}

void launch_spmv(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                 const int* istate, cudaStream_t s) {
    if (a.sell_ptr) {
        if (a.idx64) spmv_sell<int64_t>(a, x, y, b, resid, istate, s);
        else spmv_sell<int32_t>(a, x, y, b, resid, istate, s);
        return;
    }
    if (a.idx64) {
        if (a.ptr64) spmv_dispatch_l<int64_t, int64_t>(a, x, y, b, resid, istate, s);
        else spmv_dispatch_l<int64_t, int32_t>(a, x, y, b, resid, istate, s);
    } else {
        if (a.ptr64) spmv_dispatch_l<int32_t, int64_t>(a, x, y, b, resid, istate, s);
        else spmv_dispatch_l<int32_t, int32_t>(a, x, y, b, resid, istate, s);
    }
}

// ------------------------------------------------------------------------------------
// K2: fused block dot  [V_p, u]^T [u, z]   (one read of V_p, u and z per iteration)
//
// CTA = 8 warps; tile = 1024 rows; a lane owns rows {2l, 2l+1, 64+2l, 65+2l} of its warp's
// 128-row slice (two coalesced 16-B loads per column).  Columns are processed in groups of
// 8: each lane forms 8 (x2) row-partial dots, a butterfly transpose-reduction (9 shuffles
// per vector instead of 40) leaves column (lane>>2)'s warp total in lanes 4c..4c+3, and a
// per-warp shared accumulator carries it across the CTA's tiles.  Stage 2: fixed-order sum
// over warps -> per-CTA partial in global memory; the last CTA to finish (ticket counter)
// sums the partials in CTA order.  No floating-point atomics: bitwise deterministic.
// ------------------------------------------------------------------------------------
constexpr int BD_WARPS = 8;
constexpr int BD_THREADS = BD_WARPS * 32;
constexpr int BD_ROWS_W = 128;
constexpr int BD_TILE = BD_WARPS * BD_ROWS_W;
constexpr int BD_CG = 8;

__device__ __forceinline__ double bfly8(double (&a)[8], int lane) {
    // 8 values per lane -> lane holds column (lane >> 2) summed over the warp
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const bool up = lane & 16;
        const double send = up ? a[i] : a[i + 4];
        const double keep = up ? a[i + 4] : a[i];
        a[i] = keep + __shfl_xor_sync(FULL_MASK, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const bool up = lane & 8;
        const double send = up ? a[i] : a[i + 2];
        const double keep = up ? a[i + 2] : a[i];
        a[i] = keep + __shfl_xor_sync(FULL_MASK, send, 8);
    }
    {
        const bool up = lane & 4;
        const double send = up ? a[0] : a[1];
        const double keep = up ? a[1] : a[0];
        a[0] = keep + __shfl_xor_sync(FULL_MASK, send, 4);
    }
    a[0] += __shfl_xor_sync(FULL_MASK, a[0], 2);
    a[0] += __shfl_xor_sync(FULL_MASK, a[0], 1);
    return a[0];
}

template <bool GUARD>
__device__ __forceinline__ double2 bd_ld(const double* __restrict__ p, int64_t r, int64_t n) {
    if (GUARD) return ld2_guard(p, r, n);
    return __ldg(reinterpret_cast<const double2*>(p + r));
}

// one 1024-row tile for this warp's 128 rows: all column groups, accumulated into acc
template <int NV, bool GUARD>
__device__ __forceinline__ void bdot_tile(int64_t n, int p, int ncols, const double* __restrict__ V,
                                          int64_t ld, const double* __restrict__ u,
                                          const double* __restrict__ z, int64_t r0, int64_t r1,
                                          double* acc, int lane) {
    const double2 u0 = bd_ld<GUARD>(u, r0, n), u1 = bd_ld<GUARD>(u, r1, n);
    double2 z0 = make_double2(0.0, 0.0), z1 = z0;
    if (NV == 2) { z0 = bd_ld<GUARD>(z, r0, n); z1 = bd_ld<GUARD>(z, r1, n); }
    for (int cg = 0; cg < ncols; cg += BD_CG) {
        double2 va[BD_CG], vb[BD_CG];
#pragma unroll
        for (int c = 0; c < BD_CG; c++) {   // all loads first: 16 x 16 B in flight per lane
            const int j = min(cg + c, ncols - 1);
            const double* col = (j < p) ? V + (int64_t)j * ld : u;
            va[c] = bd_ld<GUARD>(col, r0, n);
            vb[c] = bd_ld<GUARD>(col, r1, n);
        }
        double au[BD_CG], az[BD_CG];
#pragma unroll
        for (int c = 0; c < BD_CG; c++) {
            const bool live = cg + c < ncols;
            const double2 v0 = va[c], v1 = vb[c];
            au[c] = live ? fma(v1.y, u1.y, fma(v1.x, u1.x, fma(v0.y, u0.y, v0.x * u0.x))) : 0.0;
            az[c] = 0.0;
            if (NV == 2) az[c] = live ? fma(v1.y, z1.y, fma(v1.x, z1.x, fma(v0.y, z0.y, v0.x * z0.x))) : 0.0;
        }
        const double su = bfly8(au, lane);
        double sz = 0.0;
        if (NV == 2) sz = bfly8(az, lane);
        const int j = cg + (lane >> 2);
        if ((lane & 3) == 0 && j < ncols) {
            acc[j] += su;
            if (NV == 2) acc[ncols + j] += sz;
        }
    }
}

template <int NV>
__global__ void __launch_bounds__(BD_THREADS, 2)
    bdot_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                const double* __restrict__ u, const double* __restrict__ z,
                double* __restrict__ part, double* __restrict__ out, unsigned* counter,
                const int* istate, const XchgDev* xc) {
    // a stopped cycle skips the work; with the cross-rank exchange every rank still joins
    // the exchange (uniform across ranks: the status word can differ between ranks)
    const bool live = running(istate);
    if (!live && !xc) return;
    extern __shared__ double sacc[];  // [BD_WARPS][NV * ncols]
    __shared__ bool s_last;
    const int ncols = p + 1;  // columns 0..p-1 of V, then u itself
    const int stride = NV * ncols;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* acc = sacc + warp * stride;
    for (int i = lane; i < stride; i += 32) acc[i] = 0.0;
    __syncwarp();

    const int64_t ntiles = live ? (n + BD_TILE - 1) / BD_TILE : 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * BD_TILE + warp * BD_ROWS_W + 2 * lane;
        const int64_t r1 = r0 + 64;
        if ((tile + 1) * BD_TILE <= n) bdot_tile<NV, false>(n, p, ncols, V, ld, u, z, r0, r1, acc, lane);
        else bdot_tile<NV, true>(n, p, ncols, V, ld, u, z, r0, r1, acc, lane);
    }
    __syncthreads();
    // stage 2a: fixed-order sum over warps -> this CTA's partial
    for (int i = threadIdx.x; i < stride; i += BD_THREADS) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < BD_WARPS; w++) s += sacc[w * stride + i];
        part[(int64_t)blockIdx.x * stride + i] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // stage 2b: last CTA sums the partials in CTA order (+ across ranks over NVLink)
    if (xc) final_reduce_xchg(part, stride, (int)gridDim.x, out, *xc);
    else final_reduce(part, stride, (int)gridDim.x, out);
    if (threadIdx.x == 0) { *counter = 0u; counter[1] += live ? 1u : 0u; }  // [1]: reductions executed
}

// ------------------------------------------------------------------------------------
// K2 (sm_100a pipeline): the same block dot with the Blackwell bulk-copy engine.
//   Persistent CTA per SM = 8 consumer warps + 1 producer warp.  Tile = 512 rows.  For each
//   tile the producer streams V_p in groups of 8 columns (8 x 4 KB cp.async.bulk copies per
//   stage, completion counted on an mbarrier with expect_tx) into a 6-stage shared-memory
//   ring (192 KB in flight per SM).  Consumer warp w owns column 8g+w of group g: lane l
//   multiplies rows l+32k (k<16) against u, z held in registers for the whole tile, one warp
//   reduction per column, and adds into a per-CTA shared accumulator that only it touches
//   for that column -> fixed order, deterministic.  Column p ("u itself") comes from the
//   registers.  Stage 2 (per-CTA partials, last CTA sums in CTA order) as in bdot_kernel.
// ------------------------------------------------------------------------------------
constexpr int BT_CONS_WARPS = 8;
constexpr int BT_THREADS = (BT_CONS_WARPS + 1) * 32;                 // column-sweep kernel
constexpr int bt_threads(int groups) { return (BT_CONS_WARPS * groups + 1) * 32; }  // tile kernel
constexpr int BT_ROWS = 512;
constexpr int BT_RPL = BT_ROWS / 32;  // rows per lane
constexpr int BT_STAGES = 6;
constexpr int BT_STAGE_DOUBLES = BT_CONS_WARPS * BT_ROWS;  // 8 columns x 512 rows = 32 KB

__device__ __forceinline__ void bdot_finish(const double* acc, int stride, double* __restrict__ part,
                                            double* __restrict__ out, unsigned* counter, bool live,
                                            const XchgDev* xc);

template <int NV, int BT_GROUPS>
__global__ void __launch_bounds__(bt_threads(BT_GROUPS), 1)
    bdot_tma_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                    const double* __restrict__ u, const double* __restrict__ z,
                    double* __restrict__ part, double* __restrict__ out, unsigned* counter,
                    const int* istate, const XchgDev* xc) {
    const bool live = running(istate);  // see bdot_kernel
    if (!live && !xc) return;
    extern __shared__ __align__(128) double smem_bt[];
    double* ring = smem_bt;                                        // [STAGES][8][512]
    double* uzslot = ring + BT_STAGES * BT_STAGE_DOUBLES;          // [2 tiles][u | z][512]
    double* acc = uzslot + 4 * BT_ROWS;                            // [NV*(p+1)]
    const int ncols = p + 1;
    const int stride = NV * ncols;
    uint64_t* full = reinterpret_cast<uint64_t*>(acc + ((BT_GROUPS * stride + 1) & ~1));
    uint64_t* empty = full + BT_STAGES;
    uint64_t* uzfull = empty + BT_STAGES;
    uint64_t* uzempty = uzfull + 2;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int warp = wid & (BT_CONS_WARPS - 1);  // column slot within a stage
    const int grp = wid / BT_CONS_WARPS;         // consumer group (BT_GROUPS = 2: stages of its parity)
    for (int i = threadIdx.x; i < BT_GROUPS * stride; i += blockDim.x) acc[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < BT_STAGES; s++) { mbar_init(full + s, 1); mbar_init(empty + s, BT_CONS_WARPS); }
        for (int s = 0; s < 2; s++) { mbar_init(uzfull + s, 1); mbar_init(uzempty + s, BT_CONS_WARPS * BT_GROUPS); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t ntiles = (n + BT_ROWS - 1) / BT_ROWS;
    const int ngroups = (ncols + BT_CONS_WARPS - 1) / BT_CONS_WARPS;
    const int64_t nk = (live && ntiles > (int64_t)blockIdx.x) ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (wid == BT_CONS_WARPS * BT_GROUPS) {
        // ---------------- producer: one elected lane issues the bulk copies ----------------
        if (lane == 0) {
            // u, z rows of tile k go to a double-buffered slot one tile ahead of tile k's V
            // stream, so the consumers never wait on a global load at a tile boundary
            auto issue_uz = [&](int64_t k) {
                const int tb = (int)(k & 1);
                const int64_t row0 = (blockIdx.x + k * gridDim.x) * BT_ROWS;
                mbar_wait(uzempty + tb, (uint32_t)(((k >> 1) & 1) ^ 1));
                if (row0 + BT_ROWS <= n) {  // full tiles only; a partial last tile is loaded directly
                    const uint32_t b = BT_ROWS * sizeof(double);
                    mbar_arrive_expect_tx(uzfull + tb, (NV == 2 ? 2 : 1) * b);
                    bulk_g2s(uzslot + (2 * tb) * BT_ROWS, u + row0, b, uzfull + tb);
                    if (NV == 2) bulk_g2s(uzslot + (2 * tb + 1) * BT_ROWS, z + row0, b, uzfull + tb);
                } else {
                    mbar_arrive(uzfull + tb);
                }
            };
            if (nk > 0) issue_uz(0);
            uint32_t it = 0;
            for (int64_t k = 0; k < nk; k++) {
                if (k + 1 < nk) issue_uz(k + 1);
                const int64_t tile = blockIdx.x + k * gridDim.x;
                const int64_t row0 = tile * BT_ROWS;
                const int64_t rows = (n - row0 < BT_ROWS) ? n - row0 : BT_ROWS;
                const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * sizeof(double));
                for (int g = 0; g < ngroups; g++, it++) {
                    const int s = it % BT_STAGES;
                    mbar_wait(empty + s, ((it / BT_STAGES) & 1) ^ 1);
                    const int c0 = g * BT_CONS_WARPS;
                    const int c1 = min(c0 + BT_CONS_WARPS, p);  // V columns only (col p = u)
                    const int nc = c1 > c0 ? c1 - c0 : 0;
                    mbar_arrive_expect_tx(full + s, (uint32_t)nc * bytes);
                    for (int c = 0; c < nc; c++)
                        bulk_g2s(ring + (size_t)s * BT_STAGE_DOUBLES + c * BT_ROWS,
                                 V + (int64_t)(c0 + c) * ld + row0, bytes, full + s);
                }
            }
        }
    } else {
        // ---------------- consumers ----------------
        uint32_t it = 0;
        for (int64_t kt = 0; kt < nk; kt++) {
            const int64_t tile = blockIdx.x + kt * gridDim.x;
            const int64_t row0 = tile * BT_ROWS;
            const bool full_tile = row0 + BT_ROWS <= n;
            const int tb = (int)(kt & 1);
            double ur[BT_RPL], zr[BT_RPL];
            mbar_wait(uzfull + tb, (uint32_t)((kt >> 1) & 1));
            if (full_tile) {
                const double* us = uzslot + (2 * tb) * BT_ROWS;
                const double* zs = uzslot + (2 * tb + 1) * BT_ROWS;
#pragma unroll
                for (int k = 0; k < BT_RPL; k++) {
                    ur[k] = us[lane + 32 * k];
                    zr[k] = NV == 2 ? zs[lane + 32 * k] : 0.0;
                }
            } else {
#pragma unroll
                for (int k = 0; k < BT_RPL; k++) {
                    const int64_t r = row0 + lane + 32 * k;
                    const bool ok = r < n;
                    ur[k] = ok ? __ldg(u + r) : 0.0;
                    zr[k] = (NV == 2 && ok) ? __ldg(z + r) : 0.0;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(uzempty + tb);
            // BT_GROUPS = 2: the two groups of 8 consumer warps take alternate stages (a stage
            // is consumed by the group of its parity), each adding into its own accumulators
            const uint32_t it0 = it;
            it += (uint32_t)ngroups;
            for (int g = BT_GROUPS == 2 ? (int)((it0 & 1u) ^ (uint32_t)grp) : 0; g < ngroups; g += BT_GROUPS) {
                const uint32_t itg = it0 + (uint32_t)g;
                const int s = itg % BT_STAGES;
                const int c = g * BT_CONS_WARPS + warp;
                mbar_wait(full + s, (itg / BT_STAGES) & 1);
                if (c < ncols) {
                    double su = 0.0, sz = 0.0;
                    if (c < p) {
                        const double* col = ring + (size_t)s * BT_STAGE_DOUBLES + warp * BT_ROWS;
                        if (full_tile) {  // no row mask: ~100 of the ~240 instructions per stage
#pragma unroll
                            for (int k = 0; k < BT_RPL; k++) {
                                const double v = col[lane + 32 * k];
                                su = fma(v, ur[k], su);
                                if (NV == 2) sz = fma(v, zr[k], sz);
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < BT_RPL; k++) {
                                double v = col[lane + 32 * k];
                                if (row0 + lane + 32 * k >= n) v = 0.0;
                                su = fma(v, ur[k], su);
                                if (NV == 2) sz = fma(v, zr[k], sz);
                            }
                        }
                    } else {  // column p is u itself
#pragma unroll
                        for (int k = 0; k < BT_RPL; k++) {
                            su = fma(ur[k], ur[k], su);
                            if (NV == 2) sz = fma(ur[k], zr[k], sz);
                        }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        su += __shfl_xor_sync(FULL_MASK, su, off);
                        if (NV == 2) sz += __shfl_xor_sync(FULL_MASK, sz, off);
                    }
                    if (lane == 0) {
                        acc[grp * stride + c] += su;
                        if (NV == 2) acc[grp * stride + ncols + c] += sz;
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
            }
        }
    }
    __syncthreads();
    if (BT_GROUPS == 2) {
        for (int i = threadIdx.x; i < stride; i += blockDim.x) acc[i] += acc[stride + i];
        __syncthreads();
    }
    bdot_finish(acc, stride, part, out, counter, live, xc);
}

// Stage 2 of the bulk-copy block dots (whole CTA, after a __syncthreads that made acc
// final): this CTA's partial to global memory, then the last K CTAs to finish (the grid is
// co-resident: one CTA per SM) each sum a contiguous slice of the 2(p+1) outputs over the
// partials in CTA order -- the same order as one finisher, K times the parallelism (c3,
// p = 300: 602 outputs x 148 partials).  With the cross-rank exchange the slices go to this
// rank's window slot and the last finisher runs the barrier and the sum over ranks
// (xchg.cuh).
__device__ __forceinline__ void bdot_finish(const double* acc, int stride, double* __restrict__ part,
                                            double* __restrict__ out, unsigned* counter, bool live,
                                            const XchgDev* xc) {
    for (int i = threadIdx.x; i < stride; i += blockDim.x) part[(int64_t)blockIdx.x * stride + i] = acc[i];
    __threadfence();
    __syncthreads();
    const int G = (int)gridDim.x;
    const int K = min(G, max(1, min(16, stride / 32)));
    __shared__ unsigned s_ticket;
    __shared__ bool s_lastf;
    if (threadIdx.x == 0) s_ticket = atomicAdd(counter, 1u);
    __syncthreads();
    const int t = (int)s_ticket;
    if (t < G - K) return;
    if (K > 1) {
        if (threadIdx.x == 0) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
            } while (v < (unsigned)G);
        }
        __syncthreads();
    }
    __threadfence();
    const unsigned call = xc ? *(volatile unsigned*)xc->calls : 0u;
    double* dst = xc ? xchg_slot(*xc, call) : out;  // [V_p^T u, u.u, V_p^T z, u.z]
    {
        const int f = t - (G - K), per = (stride + K - 1) / K;
        const int i0 = min(stride, f * per), i1 = min(stride, i0 + per);
        final_reduce_range(part, stride, G, dst, i0, i1);
    }
    if (K == 1 && !xc) {
        if (threadIdx.x == 0) { *counter = 0u; counter[1] += 1u; }  // [1]: reductions executed
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // [2]: finishers done; the last one finishes and resets the tickets
        __threadfence_system();
        s_lastf = atomicAdd(counter + 2, 1u) == (unsigned)(K - 1);
    }
    __syncthreads();
    if (!s_lastf) return;
    __threadfence();
    if (xc) xchg_finish(stride, out, *xc, call);
    if (threadIdx.x == 0) { counter[0] = 0u; counter[2] = 0u; counter[1] += live ? 1u : 0u; }
}

// ------------------------------------------------------------------------------------
// K2, column-sweep form.  The tile-at-a-time kernel above lets every CTA run through all p
// columns of one 512-row tile before the next; its CTAs drift apart, so at large p the
// grid streams from hundreds of columns (2 MB pages, 8 MB apart at c3) at once.  Here the
// CTAs sweep the columns together: a round gives CTA b the tiles r*G*S + j*G + b (j < S,
// interleaved, so the G CTAs read one contiguous range of each column), and the producer
// streams group g (8 columns) of all S tiles before group g+1.  u, z of the round's tiles
// sit in a double-buffered shared slot (bulk copies, issued when the producer reaches the
// round).  Consumer warp w owns rows 64w + 2l, +1 of every tile (16-B shared loads, u and z
// for its 2 rows), accumulates the 8 columns of the group in registers over the S tiles,
// then one butterfly transpose per group; the 8 warps' column sums meet in shared memory
// and warp g%8 adds them into the CTA accumulator in warp order.  Fixed order everywhere:
// bitwise deterministic.  Stage 2 as above (bdot_finish).
// ------------------------------------------------------------------------------------
constexpr int SW_STAGES = 4;
constexpr int SW_S = 5;  // tiles per CTA per round

static size_t bdot_sw_smem(int p, int nv) {
    const size_t stride = (size_t)nv * (p + 1);
    return (size_t)(SW_STAGES * BT_STAGE_DOUBLES + 2 * SW_S * 2 * BT_ROWS + 2 * BT_CONS_WARPS * 16) * sizeof(double) +
           ((stride + 1) & ~(size_t)1) * sizeof(double) + (2 * SW_STAGES + 4) * sizeof(uint64_t);
}

template <int NV>
__global__ void __launch_bounds__(BT_THREADS, 1)
    bdot_sw_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                   const double* __restrict__ u, const double* __restrict__ z,
                   double* __restrict__ part, double* __restrict__ out, unsigned* counter,
                   const int* istate, const XchgDev* xc) {
    const bool live = running(istate);  // see bdot_kernel
    if (!live && !xc) return;
    extern __shared__ __align__(128) double smem_sw[];
    double* ring = smem_sw;                                   // [STAGES][8][512]
    double* uzs = ring + SW_STAGES * BT_STAGE_DOUBLES;        // [2 rounds][S tiles][u | z][512]
    double* wsum = uzs + 2 * SW_S * 2 * BT_ROWS;              // [2][8 warps][16]
    double* acc = wsum + 2 * BT_CONS_WARPS * 16;              // [NV*(p+1)]
    const int ncols = p + 1;
    const int stride = NV * ncols;
    uint64_t* full = reinterpret_cast<uint64_t*>(acc + ((stride + 1) & ~1));
    uint64_t* empty = full + SW_STAGES;
    uint64_t* uzfull = empty + SW_STAGES;
    uint64_t* uzempty = uzfull + 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < stride; i += blockDim.x) acc[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < SW_STAGES; s++) { mbar_init(full + s, 1); mbar_init(empty + s, BT_CONS_WARPS); }
        for (int s = 0; s < 2; s++) { mbar_init(uzfull + s, 1); mbar_init(uzempty + s, BT_CONS_WARPS); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t ntiles = live ? (n + BT_ROWS - 1) / BT_ROWS : 0;
    const int64_t per_round = G * SW_S;
    const int64_t nrounds = (ntiles + per_round - 1) / per_round;
    const int ngroups = (ncols + 7) / 8;
    // tiles of this CTA in round r: r*G*S + j*G + b for j < nj(r)
    auto tiles_in_round = [&](int64_t r) -> int {
        const int64_t rem = ntiles - r * per_round - b;  // tiles at j*G + b < ntiles - r*G*S
        return rem <= 0 ? 0 : (int)min((int64_t)SW_S, (rem + G - 1) / G);
    };
    if (warp == BT_CONS_WARPS) {
        // ---------------- producer: one elected lane issues the bulk copies ----------------
        if (lane == 0) {
            uint32_t it = 0, kk = 0;
            for (int64_t r = 0; r < nrounds; r++) {
                const int nj = tiles_in_round(r);
                if (nj == 0) continue;
                const int slot = (int)(kk & 1);
                mbar_wait(uzempty + slot, ((kk >> 1) & 1) ^ 1);
                uint32_t uzb = 0;
                for (int j = 0; j < nj; j++)
                    if ((r * per_round + j * G + b + 1) * BT_ROWS <= n) uzb += (NV == 2 ? 2 : 1) * BT_ROWS * sizeof(double);
                mbar_arrive_expect_tx(uzfull + slot, uzb);
                for (int j = 0; j < nj; j++) {
                    const int64_t row0 = (r * per_round + j * G + b) * BT_ROWS;
                    if (row0 + BT_ROWS > n) continue;  // partial last tile: the consumers load it
                    double* dst = uzs + ((size_t)slot * SW_S + j) * 2 * BT_ROWS;
                    bulk_g2s(dst, u + row0, BT_ROWS * sizeof(double), uzfull + slot);
                    if (NV == 2) bulk_g2s(dst + BT_ROWS, z + row0, BT_ROWS * sizeof(double), uzfull + slot);
                }
                for (int g = 0; g < ngroups; g++) {
                    const int c0 = g * 8;
                    const int nc = max(0, min(8, p - c0));  // V columns only (column p = u)
                    for (int j = 0; j < nj; j++, it++) {
                        const int s = it % SW_STAGES;
                        mbar_wait(empty + s, ((it / SW_STAGES) & 1) ^ 1);
                        const int64_t row0 = (r * per_round + j * G + b) * BT_ROWS;
                        const int64_t rows = (n - row0 < BT_ROWS) ? n - row0 : BT_ROWS;
                        const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * sizeof(double));
                        mbar_arrive_expect_tx(full + s, (uint32_t)nc * bytes);
                        for (int c = 0; c < nc; c++)
                            bulk_g2s(ring + (size_t)s * BT_STAGE_DOUBLES + c * BT_ROWS,
                                     V + (int64_t)(c0 + c) * ld + row0, bytes, full + s);
                    }
                }
                kk++;
            }
        }
    } else {
        // ---------------- consumers ----------------
        const int rr = 64 * warp + 2 * lane;  // this lane's two rows within a tile
        uint32_t it = 0, kk = 0, gg = 0;      // gg: groups so far (wsum buffer parity)
        for (int64_t r = 0; r < nrounds; r++) {
            const int nj = tiles_in_round(r);
            if (nj == 0) continue;
            const int slot = (int)(kk & 1);
            const double* uzr = uzs + (size_t)slot * SW_S * 2 * BT_ROWS;
            // the partial last tile (at most one per launch): u, z straight from global memory
            int jpart = -1;
            int64_t prow0 = 0;
            double pu0 = 0.0, pu1 = 0.0, pz0 = 0.0, pz1 = 0.0;
            for (int j = 0; j < nj; j++) {
                const int64_t row0 = (r * per_round + j * G + b) * BT_ROWS;
                if (row0 + BT_ROWS > n) {
                    jpart = j;
                    prow0 = row0;
                    const int64_t r0 = row0 + rr;
                    if (r0 < n) { pu0 = __ldg(u + r0); if (NV == 2) pz0 = __ldg(z + r0); }
                    if (r0 + 1 < n) { pu1 = __ldg(u + r0 + 1); if (NV == 2) pz1 = __ldg(z + r0 + 1); }
                }
            }
            mbar_wait(uzfull + slot, (kk >> 1) & 1);
            for (int g = 0; g < ngroups; g++) {
                const int c0 = g * 8;
                const int nvc = max(0, min(8, p - c0));  // V columns in this group
                const int cu = p - c0;                   // column p (u itself) if 0 <= cu < 8
                double au[8], az[8];
#pragma unroll
                for (int c = 0; c < 8; c++) { au[c] = 0.0; az[c] = 0.0; }
                for (int j = 0; j < nj; j++, it++) {
                    const int s = it % SW_STAGES;
                    double u0, u1, z0 = 0.0, z1 = 0.0;
                    const bool part_tile = (j == jpart);
                    if (part_tile) {
                        u0 = pu0; u1 = pu1; z0 = pz0; z1 = pz1;
                    } else {
                        const double2 uu = *reinterpret_cast<const double2*>(uzr + (size_t)j * 2 * BT_ROWS + rr);
                        u0 = uu.x; u1 = uu.y;
                        if (NV == 2) {
                            const double2 zz = *reinterpret_cast<const double2*>(uzr + (size_t)j * 2 * BT_ROWS + BT_ROWS + rr);
                            z0 = zz.x; z1 = zz.y;
                        }
                    }
                    mbar_wait(full + s, (it / SW_STAGES) & 1);
                    const double* st = ring + (size_t)s * BT_STAGE_DOUBLES + rr;
                    const bool m0 = !part_tile || prow0 + rr < n, m1 = !part_tile || prow0 + rr + 1 < n;
#pragma unroll
                    for (int c = 0; c < 8; c++) {
                        double2 v;
                        if (c < nvc) {
                            v = *reinterpret_cast<const double2*>(st + c * BT_ROWS);
                            if (part_tile) { v.x = m0 ? v.x : 0.0; v.y = m1 ? v.y : 0.0; }
                        } else if (c == cu) {
                            v = make_double2(u0, u1);
                        } else {
                            continue;
                        }
                        au[c] = fma(v.y, u1, fma(v.x, u0, au[c]));
                        if (NV == 2) az[c] = fma(v.y, z1, fma(v.x, z0, az[c]));
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + s);
                }
                // column c0 + (lane >> 2) summed over this warp's rows, in lanes 4c..4c+3
                const double su = bfly8(au, lane);
                const double sz = NV == 2 ? bfly8(az, lane) : 0.0;
                double* ws = wsum + (gg++ & 1) * BT_CONS_WARPS * 16;
                if ((lane & 3) == 0) {
                    ws[warp * 16 + (lane >> 2)] = su;
                    ws[warp * 16 + 8 + (lane >> 2)] = sz;
                }
                named_barrier(1, BT_CONS_WARPS * 32);
                if (warp == (g & 7) && lane < 8 * NV) {  // lanes 0-7: V^T u column sums, 8-15: V^T z
                    const int c = lane & 7, col = c0 + c;
                    if (col < ncols) {
                        double t = 0.0;
#pragma unroll
                        for (int w = 0; w < BT_CONS_WARPS; w++) t += ws[w * 16 + lane];
                        acc[(lane >> 3) * ncols + col] += t;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(uzempty + slot);
            kk++;
        }
    }
    __syncthreads();
    bdot_finish(acc, stride, part, out, counter, live, xc);
}

int bdot_grid_size(int64_t n, int num_sms) {
    const int64_t ntiles = (n + BD_TILE - 1) / BD_TILE;
    int64_t g = (int64_t)num_sms * 2;
    if (g > ntiles) g = ntiles;
    // also >= the bulk-copy kernels' grid (one CTA per 512-row tile, at most one per SM): with
    // 1024-row register tiles alone, n in (75K, 151K) left the bulk-copy kernel out
    const int64_t tg = std::min<int64_t>((n + BT_ROWS - 1) / BT_ROWS, num_sms);
    if (g < tg) g = tg;
    if (g < 1) g = 1;
    return (int)g;
}

// consumer groups of the tile kernel: two groups of 8 warps on alternate stages from four
// column groups per tile on (p >= 24; 4 consumer warps per scheduler instead of 2: c4 p = 50
// isolated 992 -> 955 us = 7.3 TB/s, bench block dot 102.6 -> 100.8 ms per step).  With fewer
// column groups the second warp group idles or unbalances the tile (p = 10: 310 -> 330 us;
// p = 16 / 20: 393 / 434 vs 397 / 441 us; p = 24 / 32: 530 / 665 -> 509 / 631 us,
// profiles/r2/c42)
static int bdot_tma_groups(int p) {
    static int force = -1;  // A/B hook: IGS_BDOT_GROUPS=1 keeps one consumer group at every p
    if (force < 0) { const char* e = std::getenv("IGS_BDOT_GROUPS"); force = e ? std::atoi(e) : 0; }
    if (force == 1) return 1;
    return p + 1 > 3 * BT_CONS_WARPS ? 2 : 1;
}

static size_t bdot_tma_smem(int p, int nv) {
    const size_t stride = (size_t)nv * (p + 1);
    return (size_t)(BT_STAGES * BT_STAGE_DOUBLES + 4 * BT_ROWS) * sizeof(double) +
           ((bdot_tma_groups(p) * stride + 1) & ~(size_t)1) * sizeof(double) + (2 * BT_STAGES + 4) * sizeof(uint64_t);
}

static size_t bdot_smem(int p, int nv) { return (size_t)BD_WARPS * nv * (p + 1) * sizeof(double); }

void launch_block_dot(int64_t n, int p, const double* V, int64_t ld, const double* u,
                      const double* z, double* out, double* part, unsigned* counter, int grid,
                      const int* istate, cudaStream_t s, const XchgDev* xc) {
    const int nv = z ? 2 : 1;
    // sm_100a bulk-copy pipeline when V columns are 16-B aligned with an even ld and the
    // accumulators fit next to the 192 KB ring; the register kernel otherwise
    const size_t tsmem = bdot_tma_smem(p, nv);
    if (p > 0 && (ld % 2) == 0 && ((uintptr_t)V % 16) == 0 && tsmem <= 227 * 1024 && n >= BT_ROWS) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t ntiles = (n + BT_ROWS - 1) / BT_ROWS;
        const int tg = (int)(ntiles < sms ? ntiles : sms);
        // the column sweep from p = 96 on (c3 p = 300: 6.39 -> 6.75 TB/s; at p = 10-75 the
        // tile kernel is ahead: c4 p = 25 6.92 vs 5.79; profiles/r2/bdot_sweep_ab.md);
        // and below p = 8 (one column group: the tile kernel's two u, z slots allow a single
        // tile of lookahead there -- c4 p = 1 / 5: 203 / 231 -> 148 / 177 us isolated, 0.3 ms of the
        // 242 ms bench step in an alternating A/B, profiles/r2/c26);
        // IGS_BDOT_SW_MIN_P moves the upper switch (A/B and test hook; it also disables the
        // small-p use when above 1000)
        static int sw_min_p = -1;
        if (sw_min_p < 0) {
            const char* e = std::getenv("IGS_BDOT_SW_MIN_P");
            sw_min_p = e ? std::atoi(e) : 96;
        }
        const size_t wsmem = bdot_sw_smem(p, nv);
        const bool sweep = p >= sw_min_p || (p < 8 && sw_min_p <= 1000);
        if (tg <= grid && sweep && wsmem <= 227 * 1024) {
            if (nv == 2) {
                cudaFuncSetAttribute(bdot_sw_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem);
                bdot_sw_kernel<2><<<tg, BT_THREADS, wsmem, s>>>(n, p, V, ld, u, z, part, out, counter, istate, xc);
            } else {
                cudaFuncSetAttribute(bdot_sw_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem);
                bdot_sw_kernel<1><<<tg, BT_THREADS, wsmem, s>>>(n, p, V, ld, u, z, part, out, counter, istate, xc);
            }
            return;
        }
        if (tg <= grid) {
#define IGS_BT_LAUNCH(NVV, GG)                                                                                    \
    do {                                                                                                          \
        cudaFuncSetAttribute(bdot_tma_kernel<NVV, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem); \
        bdot_tma_kernel<NVV, GG><<<tg, bt_threads(GG), tsmem, s>>>(n, p, V, ld, u, z, part, out, counter, istate, xc); \
    } while (0)
            const int gg = bdot_tma_groups(p);
            if (nv == 2) { if (gg == 2) IGS_BT_LAUNCH(2, 2); else IGS_BT_LAUNCH(2, 1); }
            else { if (gg == 2) IGS_BT_LAUNCH(1, 2); else IGS_BT_LAUNCH(1, 1); }
#undef IGS_BT_LAUNCH
            return;
        }
    }
    const size_t smem = bdot_smem(p, nv);
    if (nv == 2) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(bdot_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        bdot_kernel<2><<<grid, BD_THREADS, smem, s>>>(n, p, V, ld, u, z, part, out, counter, istate, xc);
    } else {
        if (smem > 48 * 1024) cudaFuncSetAttribute(bdot_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        bdot_kernel<1><<<grid, BD_THREADS, smem, s>>>(n, p, V, ld, u, z, part, out, counter, istate, xc);
    }
}

// ------------------------------------------------------------------------------------
// K5: fused update with lagged normalisation (one read of V_p)
//   w = u - V_p alpha  (HAS_ALPHA; Alg. 3 Step 10 "Jacobi iteration")  or w = u
//   v = w / gamma                                     (Step 11 / Alg. 2 Step 7)
//   u' = z / gamma - (V_p beta[:p] + v beta[p])       (Step 13)
// Each thread owns two consecutive rows (16-B loads); columns unrolled 8-deep.
// ------------------------------------------------------------------------------------
constexpr int UP_THREADS = 256;

template <bool HAS_ALPHA>
__global__ void __launch_bounds__(UP_THREADS)
    update_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                  const double* u, const double* __restrict__ z,
                  const double* __restrict__ alpha, const double* __restrict__ beta,
                  const double* __restrict__ gamma_dev, double* v_out, double* u_next,
                  const int* istate, int it, int default_mode, const double* __restrict__ zdiv_dev) {
    extern __shared__ double coef[];  // alpha[p] | beta[p+1]
    int mode = default_mode;
    if (istate) {
        const volatile int* vs = istate;
        mode = (vs[ST_MODE_IT] == it) ? vs[ST_MODE] : 0;
        mode &= default_mode;  // never write u' without a u' buffer
    }
    if (mode == 0) return;
    const bool want_next = (mode & 2) != 0;
    double* sa = coef;
    double* sb = coef + p;
    if (HAS_ALPHA)
        for (int j = threadIdx.x; j < p; j += blockDim.x) sa[j] = alpha[j];
    if (want_next)
        for (int j = threadIdx.x; j <= p; j += blockDim.x) sb[j] = beta[j];
    __syncthreads();
    const double gamma = *gamma_dev;
    const double zdiv = zdiv_dev ? *zdiv_dev : gamma;  // z / gamma (Arnoldi) or z / 1 (QR)
    // grid-stride form; launch_update gives every CTA one tile
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; r < n;
         r += (int64_t)gridDim.x * blockDim.x * 2) {
        const bool pair = (r + 1 < n);
        // u and z first: their latency overlaps the column loop
        const double2 uu = ld2_guard(u, r, n);
        const double2 zz = want_next ? ld2_guard(z, r, n) : make_double2(0.0, 0.0);
        double2 t1 = make_double2(0.0, 0.0), t2 = make_double2(0.0, 0.0);
        if (HAS_ALPHA || want_next) {
            int j = 0;
            if (pair) {
                for (; j + 8 <= p; j += 8) {
                    double2 v[8];
#pragma unroll
                    for (int c = 0; c < 8; c++) v[c] = __ldg(reinterpret_cast<const double2*>(V + (int64_t)(j + c) * ld + r));
#pragma unroll
                    for (int c = 0; c < 8; c++) {
                        if (HAS_ALPHA) { t1.x = fma(v[c].x, sa[j + c], t1.x); t1.y = fma(v[c].y, sa[j + c], t1.y); }
                        if (want_next) { t2.x = fma(v[c].x, sb[j + c], t2.x); t2.y = fma(v[c].y, sb[j + c], t2.y); }
                    }
                }
                if (j < p) {  // the last p mod 8 columns: loads issued together, then the FMAs in order
                    double2 v[8];
#pragma unroll
                    for (int c = 0; c < 8; c++)
                        v[c] = (j + c < p) ? __ldg(reinterpret_cast<const double2*>(V + (int64_t)(j + c) * ld + r))
                                           : make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < 8; c++) {
                        if (j + c >= p) break;
                        if (HAS_ALPHA) { t1.x = fma(v[c].x, sa[j + c], t1.x); t1.y = fma(v[c].y, sa[j + c], t1.y); }
                        if (want_next) { t2.x = fma(v[c].x, sb[j + c], t2.x); t2.y = fma(v[c].y, sb[j + c], t2.y); }
                    }
                    j = p;
                }
            }
            for (; j < p; j++) {
                const double2 v = ld2_guard(V + (int64_t)j * ld, r, n);
                if (HAS_ALPHA) { t1.x = fma(v.x, sa[j], t1.x); t1.y = fma(v.y, sa[j], t1.y); }
                if (want_next) { t2.x = fma(v.x, sb[j], t2.x); t2.y = fma(v.y, sb[j], t2.y); }
            }
        }
        double2 w = uu;
        if (HAS_ALPHA) { w.x = uu.x - t1.x; w.y = uu.y - t1.y; }
        double2 v;
        v.x = w.x / gamma;
        v.y = w.y / gamma;
        if (want_next) {
            const double bp = sb[p];
            double2 un;
            un.x = zz.x / zdiv - fma(v.x, bp, t2.x);
            un.y = zz.y / zdiv - fma(v.y, bp, t2.y);
            u_next[r] = un.x;
            if (pair) u_next[r + 1] = un.y;
        }
        if (mode & 1) {
            v_out[r] = v.x;
            if (pair) v_out[r + 1] = v.y;
        }
    }
}

// ------------------------------------------------------------------------------------
// Alg. 2 two-reduce: the first fused update (Steps 7-13, as update_kernel, bitwise the same
// v and u') fused with the second sweep's block dot r2 = V_{p+1}^T u' (Step 14)
// and u'.u'.  Per 512-row tile each thread (two rows) computes v, u' in one pass over V_p
// (HBM), writes them, then passes over the same V_p rows again -- an L2 re-read of the tile
// the CTA just streamed -- for the p + 2 dots; 8 columns per butterfly (bfly8), per-warp
// accumulators in shared memory in tile order, per-CTA partials summed by the last CTA in CTA
// order (+ across ranks over NVLink when xc != nullptr).  One HBM read of V_p instead of two.
// out = [V_p^T u', v.u', u'.u'] (the layout of launch_block_dot(p + 1, u', NULL)).
// ------------------------------------------------------------------------------------
constexpr int UD_THREADS = 256, UD_WARPS = UD_THREADS / 32, UD_TILE = 2 * UD_THREADS;

template <bool HAS_ALPHA>
__global__ void __launch_bounds__(UD_THREADS)
    update_dot_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                      const double* u, const double* __restrict__ z,
                      const double* __restrict__ alpha, const double* __restrict__ beta,
                      const double* __restrict__ gamma_dev, double* v_out, double* u_next,
                      const int* istate, int it, double* __restrict__ part, double* out,
                      unsigned* counter, const XchgDev* xc) {
    extern __shared__ double sdyn[];  // alpha[p] | beta[p+1] | acc[UD_WARPS][p+2]
    __shared__ bool s_last;
    bool live = true;
    if (istate) {
        const volatile int* vs = istate;
        const int mode = (vs[ST_MODE_IT] == it) ? vs[ST_MODE] : 0;
        live = (mode & 3) == 3;  // the second sweep runs only after a full update
    }
    if (!live && !xc) return;  // with the exchange every rank joins it (bdot_kernel)
    const int nd = p + 2;
    double* sa = sdyn;
    double* sb = sdyn + p;
    double* acc = sb + p + 1 + (threadIdx.x >> 5) * nd;
    const int lane = threadIdx.x & 31;
    if (HAS_ALPHA)
        for (int j = threadIdx.x; j < p; j += blockDim.x) sa[j] = alpha[j];
    for (int j = threadIdx.x; j <= p; j += blockDim.x) sb[j] = beta[j];
    for (int j = lane; j < nd; j += 32) acc[j] = 0.0;
    __syncthreads();
    const double gamma = *gamma_dev;
    const int64_t ntiles = live ? (n + UD_TILE - 1) / UD_TILE : 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r = tile * UD_TILE + 2 * threadIdx.x;
        const bool in = r < n, pair = r + 1 < n;
        // ---- pass 1: exactly update_kernel's arithmetic for rows r, r+1
        double2 t1 = make_double2(0.0, 0.0), t2 = make_double2(0.0, 0.0);
        int j = 0;
        if (pair) {
            for (; j + 8 <= p; j += 8) {
                double2 v[8];
#pragma unroll
                for (int c = 0; c < 8; c++) v[c] = __ldg(reinterpret_cast<const double2*>(V + (int64_t)(j + c) * ld + r));
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    if (HAS_ALPHA) { t1.x = fma(v[c].x, sa[j + c], t1.x); t1.y = fma(v[c].y, sa[j + c], t1.y); }
                    t2.x = fma(v[c].x, sb[j + c], t2.x); t2.y = fma(v[c].y, sb[j + c], t2.y);
                }
            }
        }
        if (in) {
            for (; j < p; j++) {
                const double2 v = ld2_guard(V + (int64_t)j * ld, r, n);
                if (HAS_ALPHA) { t1.x = fma(v.x, sa[j], t1.x); t1.y = fma(v.y, sa[j], t1.y); }
                t2.x = fma(v.x, sb[j], t2.x); t2.y = fma(v.y, sb[j], t2.y);
            }
        }
        double2 vv = make_double2(0.0, 0.0), un = make_double2(0.0, 0.0);
        if (in) {
            const double2 uu = ld2_guard(u, r, n);
            double2 w = uu;
            if (HAS_ALPHA) { w.x = uu.x - t1.x; w.y = uu.y - t1.y; }
            vv.x = w.x / gamma;
            vv.y = w.y / gamma;
            const double2 zz = ld2_guard(z, r, n);
            const double bp = sb[p];
            un.x = zz.x / gamma - fma(vv.x, bp, t2.x);
            un.y = zz.y / gamma - fma(vv.y, bp, t2.y);
            if (!pair) { vv.y = 0.0; un.y = 0.0; }
            u_next[r] = un.x;
            if (pair) u_next[r + 1] = un.y;
            v_out[r] = vv.x;
            if (pair) v_out[r + 1] = vv.y;
        }
        // ---- pass 2: the p + 2 dots of the tile, 8 columns per butterfly (L2 re-read of V_p)
        for (int cb = 0; cb < nd; cb += 8) {
            double a[8];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int col = cb + c;
                double2 x = make_double2(0.0, 0.0);
                if (col < p) x = in ? ld2_guard(V + (int64_t)col * ld, r, n) : x;
                else if (col == p) x = vv;
                else if (col == p + 1) x = un;
                a[c] = fma(x.y, un.y, x.x * un.x);
            }
            const double t = bfly8(a, lane);  // lane holds column cb + (lane >> 2)
            const int col = cb + (lane >> 2);
            if ((lane & 3) == 0 && col < nd) acc[col] += t;
        }
    }
    __syncthreads();
    // per-CTA partial: warps summed in warp order
    for (int j = threadIdx.x; j < nd; j += blockDim.x) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < UD_WARPS; w++) t += sb[p + 1 + w * nd + j];
        part[(int64_t)blockIdx.x * nd + j] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (xc) final_reduce_xchg(part, nd, (int)gridDim.x, out, *xc);
    else final_reduce(part, nd, (int)gridDim.x, out);
    if (threadIdx.x == 0) { *counter = 0u; counter[1] += live ? 1u : 0u; }
}

// The same fused update + second-sweep dot with the V_p tile resident in shared memory:
// 1 producer warp bulk-copies 128-row x p-column tiles (one 1-KB copy per column) into a
// 2-buffer ring; consumer threads (one per tile row) compute v, u' from shared memory
// (update_kernel's FMA sequence: bitwise the same v, u'), then all 8 consumer warps form the
// p + 2 dots from the same shared tile (8 columns per butterfly, R / 32 rows per lane).  One HBM
// read of V_p and no L2 re-read; p <= update_dot_tma_max_p() (two tiles in 227 KB).
constexpr int UT_CONS = 8, UT_THREADS = (UT_CONS + 1) * 32;
#ifndef UT_RSTEP
#define UT_RSTEP 32   // 128: only 256- or 128-row tiles (A/B build)
#endif

// tile rows R (128 .. 256 in steps of UT_RSTEP) x (p V columns + u + z), two tiles in flight
size_t update_dot_tma_smem(int p, int R) {
    return (size_t)2 * (p + 2) * R * sizeof(double) +
           (size_t)(2 * p + 1 + 2 * R + UT_CONS * (p + 2)) * sizeof(double) + 4 * sizeof(uint64_t);
}

int update_dot_tma_rows(int p) {  // the tallest tile (multiple of 32 rows) of which two fit; 0: none
    for (int R = 256; R >= 128; R -= UT_RSTEP)
        if (update_dot_tma_smem(p, R) <= 227 * 1024) return R;
    return 0;
}

template <bool HAS_ALPHA>
__global__ void __launch_bounds__(UT_THREADS, 1)
    update_dot_tma_kernel(int64_t n, int p, int R, const double* __restrict__ V, int64_t ld,
                          const double* u, const double* __restrict__ z,
                          const double* __restrict__ alpha, const double* __restrict__ beta,
                          const double* __restrict__ gamma_dev, double* v_out, double* u_next,
                          const int* istate, int it, double* __restrict__ part, double* out,
                          unsigned* counter, const XchgDev* xc) {
    extern __shared__ __align__(16) double usm[];
    __shared__ bool s_last;
    bool live = true;
    if (istate) {
        const volatile int* vs = istate;
        const int mode = (vs[ST_MODE_IT] == it) ? vs[ST_MODE] : 0;
        live = (mode & 3) == 3;
    }
    if (!live && !xc) return;  // with the exchange every rank joins it (bdot_kernel)
    const int nd = p + 2, tcols = p + 2;  // tile columns: V_p | u | z
    double* buf = usm;                                // [2][tcols][R]
    double* sa = buf + (size_t)2 * tcols * R;         // [p]
    double* sb = sa + p;                              // [p + 1]
    double* s_v = sb + p + 1;                         // [R]
    double* s_un = s_v + R;                           // [R]
    double* acc = s_un + R;                           // [UT_CONS][nd]
    uint64_t* full = reinterpret_cast<uint64_t*>(acc + UT_CONS * nd);
    uint64_t* empty = full + 2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int b = 0; b < 2; b++) { mbar_init(full + b, 1); mbar_init(empty + b, UT_CONS); }
        mbar_fence_init();
    }
    if (HAS_ALPHA)
        for (int j = tid; j < p; j += blockDim.x) sa[j] = alpha[j];
    for (int j = tid; j <= p; j += blockDim.x) sb[j] = beta[j];
    for (int j = tid; j < UT_CONS * nd; j += blockDim.x) acc[j] = 0.0;
    __syncthreads();
    const double gamma = *gamma_dev;
    const int64_t ntiles = (n + R - 1) / R;
    const int64_t nk = (live && blockIdx.x < ntiles) ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp == UT_CONS) {
        // ---------------- producer warp: one bulk copy per column (and u, z) and tile ----------
        for (int64_t k = 0; k < nk; k++) {
            const int b = (int)(k & 1);
            const int64_t row0 = (blockIdx.x + k * gridDim.x) * R;
            const int64_t rows = (n - row0 < R) ? n - row0 : R;
            const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * sizeof(double));
            mbar_wait(empty + b, (uint32_t)(((k >> 1) & 1) ^ 1));
            if (lane == 0) mbar_arrive_expect_tx(full + b, (uint32_t)tcols * bytes);
            __syncwarp();
            double* dst = buf + (size_t)b * tcols * R;
            for (int j = lane; j < tcols; j += 32) {
                const double* src = j < p ? V + (int64_t)j * ld + row0 : (j == p ? u + row0 : z + row0);
                bulk_g2s(dst + (size_t)j * R, src, bytes, full + b);
            }
        }
    } else {
        // ---------------- consumers ----------------
        for (int64_t k = 0; k < nk; k++) {
            const int b = (int)(k & 1);
            const int64_t row0 = (blockIdx.x + k * gridDim.x) * R;
            const double* tb = buf + (size_t)b * tcols * R;
            mbar_wait(full + b, (uint32_t)((k >> 1) & 1));
            if (tid < R) {  // pass 1: row r -- update_kernel's per-row FMA sequence (bitwise equal)
                const int64_t r = row0 + tid;
                double vv = 0.0, un = 0.0;
                if (r < n) {
                    double t1 = 0.0, t2 = 0.0;
#pragma unroll 8
                    for (int j = 0; j < p; j++) {
                        const double v = tb[(size_t)j * R + tid];
                        if (HAS_ALPHA) t1 = fma(v, sa[j], t1);
                        t2 = fma(v, sb[j], t2);
                    }
                    const double uu = tb[(size_t)p * R + tid], zz = tb[(size_t)(p + 1) * R + tid];
                    const double w = HAS_ALPHA ? uu - t1 : uu;
                    vv = w / gamma;
                    un = zz / gamma - fma(vv, sb[p], t2);
                    u_next[r] = un;
                    v_out[r] = vv;
                }
                s_v[tid] = vv;
                s_un[tid] = un;
            }
            named_barrier(1, UT_CONS * 32);
            // pass 2: the p + 2 dots of the tile (rows beyond n carry u' = 0 and are skipped)
            const int64_t nrows = n - row0;
            const int rpl = R / 32;  // rows lane, lane + 32, ... (conflict-free shared loads)
            for (int cb = 8 * warp; cb < nd; cb += 8 * UT_CONS) {
                double a[8];
#pragma unroll
                for (int c = 0; c < 8; c++) a[c] = 0.0;
                for (int q = 0; q < rpl; q++) {
                    const int rr = lane + 32 * q;
                    if (rr < nrows) {
                        const double w = s_un[rr];
#pragma unroll
                        for (int c = 0; c < 8; c++) {
                            const int col = cb + c;
                            if (col < nd) {
                                const double* src = col < p ? tb + (size_t)col * R : (col == p ? s_v : s_un);
                                a[c] = fma(src[rr], w, a[c]);
                            }
                        }
                    }
                }
                const double t = bfly8(a, lane);
                const int colx = cb + (lane >> 2);
                if ((lane & 3) == 0 && colx < nd) acc[warp * nd + colx] += t;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + b);
            named_barrier(1, UT_CONS * 32);  // s_v / s_un are rewritten by the next tile
        }
    }
    __syncthreads();
    for (int j = tid; j < nd; j += blockDim.x) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < UT_CONS; w++) t += acc[w * nd + j];
        part[(int64_t)blockIdx.x * nd + j] = t;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (xc) final_reduce_xchg(part, nd, (int)gridDim.x, out, *xc);
    else final_reduce(part, nd, (int)gridDim.x, out);
    if (tid == 0) { *counter = 0u; counter[1] += live ? 1u : 0u; }
}

void launch_update_dot_tma(int64_t n, int p, const double* V, int64_t ld, const double* u, const double* z,
                           const double* alpha, const double* beta, const double* gamma_dev, double* v_out,
                           double* u_next, const int* istate, int it, double* part, double* out,
                           unsigned* counter, int grid, const XchgDev* xc, cudaStream_t s) {
    const int R = update_dot_tma_rows(p);
    const size_t smem = update_dot_tma_smem(p, R);
    if (alpha) {
        cudaFuncSetAttribute(update_dot_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        update_dot_tma_kernel<true><<<grid, UT_THREADS, smem, s>>>(n, p, R, V, ld, u, z, alpha, beta, gamma_dev, v_out,
                                                                   u_next, istate, it, part, out, counter, xc);
    } else {
        cudaFuncSetAttribute(update_dot_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        update_dot_tma_kernel<false><<<grid, UT_THREADS, smem, s>>>(n, p, R, V, ld, u, z, alpha, beta, gamma_dev, v_out,
                                                                    u_next, istate, it, part, out, counter, xc);
    }
}

int update_dot_grid(int64_t n, int num_sms) {
    const int64_t ntiles = (n + UD_TILE - 1) / UD_TILE;
    const int mult = 4;  // CTAs per SM
    int64_t g = (int64_t)num_sms * mult;
    if (g > ntiles) g = ntiles;
    return (int)(g < 1 ? 1 : g);
}

size_t update_dot_smem(int p) { return (size_t)(2 * p + 1 + UD_WARPS * (p + 2)) * sizeof(double); }

void launch_update_dot(int64_t n, int p, const double* V, int64_t ld, const double* u, const double* z,
                       const double* alpha, const double* beta, const double* gamma_dev, double* v_out,
                       double* u_next, const int* istate, int it, double* part, double* out,
                       unsigned* counter, int grid, const XchgDev* xc, cudaStream_t s) {
    const size_t smem = update_dot_smem(p);
    if (alpha) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(update_dot_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        update_dot_kernel<true><<<grid, UD_THREADS, smem, s>>>(n, p, V, ld, u, z, alpha, beta, gamma_dev, v_out,
                                                               u_next, istate, it, part, out, counter, xc);
    } else {
        if (smem > 48 * 1024) cudaFuncSetAttribute(update_dot_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        update_dot_kernel<false><<<grid, UD_THREADS, smem, s>>>(n, p, V, ld, u, z, alpha, beta, gamma_dev, v_out,
                                                                u_next, istate, it, part, out, counter, xc);
    }
}

void launch_update(int64_t n, int p, const double* V, int64_t ld, const double* u,
                   const double* z, const double* alpha, const double* beta,
                   const double* gamma_dev, double* v_out, double* u_next, const int* istate,
                   int it, cudaStream_t s, const double* zdiv_dev) {
    const int64_t nthreads = (n + 1) / 2;
    // one 512-row tile per CTA: capping the grid at the resident CTAs (grid-stride, prologue
    // once per CTA) measured slower beyond p ~ 10 (c4 399.5 vs 403.7 it/s)
    const unsigned blocks = (unsigned)((nthreads + UP_THREADS - 1) / UP_THREADS);
    if (blocks == 0) return;
    const size_t smem = (size_t)(2 * p + 1) * sizeof(double);
    const int dmode = 1 | (u_next ? 2 : 0);
    if (alpha) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(update_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        update_kernel<true><<<blocks, UP_THREADS, smem, s>>>(n, p, V, ld, u, z, alpha, beta, gamma_dev, v_out, u_next, istate, it, dmode, zdiv_dev);
    } else {
        if (smem > 48 * 1024) cudaFuncSetAttribute(update_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        update_kernel<false><<<blocks, UP_THREADS, smem, s>>>(n, p, V, ld, u, z, alpha, beta, gamma_dev, v_out, u_next, istate, it, dmode, zdiv_dev);
    }
}

// x += V[:, :p] y   (p = istate[ST_PDONE])
__global__ void __launch_bounds__(UP_THREADS)
    xupdate_kernel(int64_t n, const double* __restrict__ V, int64_t ld,
                   const double* __restrict__ y, double* x, const int* istate) {
    extern __shared__ double sy[];
    const int p = istate[ST_PDONE];
    for (int j = threadIdx.x; j < p; j += blockDim.x) sy[j] = y[j];
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n || p == 0) return;
    double t = 0.0;
    int j = 0;
    for (; j + 8 <= p; j += 8) {
        double v[8];
#pragma unroll
        for (int c = 0; c < 8; c++) v[c] = __ldg(V + (int64_t)(j + c) * ld + r);
#pragma unroll
        for (int c = 0; c < 8; c++) t = fma(v[c], sy[j + c], t);
    }
    for (; j < p; j++) t = fma(__ldg(V + (int64_t)j * ld + r), sy[j], t);
    x[r] = x[r] + t;
}

void launch_xupdate(int64_t n, const double* V, int64_t ld, const double* y, double* x,
                    const int* istate, int pmax, cudaStream_t s) {
    const unsigned blocks = (unsigned)((n + UP_THREADS - 1) / UP_THREADS);
    if (blocks == 0) return;
    xupdate_kernel<<<blocks, UP_THREADS, (size_t)(pmax + 1) * sizeof(double), s>>>(n, V, ld, y, x, istate);
}

// ------------------------------------------------------------------------------------
// K4: the small step (one CTA, replicated on every rank from the bit-identical reduced
// dot vector).  Split in two kernels:
//   crit  (main stream)  -- exactly what the fused update needs: gamma, the update
//                           coefficients alpha = r2 and beta = r1, L[p,:p], mode bits;
//   tail  (side stream)  -- what only the Hessenberg/least-squares state needs: r3, the H
//                           column, Givens, residual, convergence/breakdown status, hp.
// For Alg. 3 the (I+L)^{-1} solve (Step 5) only feeds H (Step 14), so it runs in the tail,
// overlapped with the update kernel; for Alg. 2 (one sweep) r1 = (I+L)^{-1} c is on the
// critical path.  Deterministic block reductions; blocked forward substitution.
// ------------------------------------------------------------------------------------
constexpr int SS_THREADS = 512;

__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL_MASK, v, off);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(FULL_MASK, t, off);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// x <- (I + L)^{-1} x in shared memory: forward substitution blocked by 32.
// Row i still subtracts L[i,j] x_j for j = 0, 1, 2, ... in natural order; warp 0 solves each
// 32x32 diagonal block with shuffles, then every thread updates its trailing rows with 32
// independent loads in flight.
#ifndef TRISOLVE_LOOKAHEAD
#define TRISOLVE_LOOKAHEAD 1
#endif
__device__ __forceinline__ void trisolve_smem(int order, const double* __restrict__ L, int ldl, double* x) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if TRISOLVE_LOOKAHEAD
    // Lookahead schedule (blockDim >= 96): at step k warp 1 applies block k-1 to the rows of
    // block k only while warp 0 loads block k's diagonal L entries; then warp 0 runs the
    // 32-step shuffle chain.  Meanwhile warps 2.. apply block k-1 to the rows below block k.
    // Every row still receives the blocks' contributions in ascending order with the same
    // FMA sequence as the right-looking loop (#else), so the result is bitwise the same; the
    // step's critical path loses the second dependent L2 round trip.
    __syncthreads();
    for (int kb = 0; kb < order; kb += 32) {
        const int nb = min(32, order - kb);
        if (warp <= 1) {
            const int i = kb + lane;
            if (warp == 1) {
                if (kb > 0 && lane < nb) {  // block k-1 (full: only the last block is partial)
                    double lv[32];
#pragma unroll
                    for (int j = 0; j < 32; j++) lv[j] = __ldcg(L + i + (int64_t)(kb - 32 + j) * ldl);
                    double sacc = x[i];
#pragma unroll
                    for (int j = 0; j < 32; j++) sacc = sacc - lv[j] * x[kb - 32 + j];
                    x[i] = sacc;
                }
                named_barrier(2, 64);
            } else {
                const bool mine = lane < nb;
                double lrow[32];
#pragma unroll
                for (int j = 0; j < 32; j++)
                    lrow[j] = (mine && j < lane) ? __ldcg(L + (kb + lane) + (int64_t)(kb + j) * ldl) : 0.0;
                named_barrier(2, 64);
                double xi = mine ? x[kb + lane] : 0.0;
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    const double xj = __shfl_sync(FULL_MASK, xi, j);
                    if (j < lane) xi = xi - lrow[j] * xj;
                }
                if (mine) x[kb + lane] = xi;
            }
        } else if (kb > 0) {
            for (int i = kb + nb + (int)threadIdx.x - 64; i < order; i += (int)blockDim.x - 64) {
                double lv[32];
#pragma unroll
                for (int j = 0; j < 32; j++) lv[j] = __ldcg(L + i + (int64_t)(kb - 32 + j) * ldl);
                double sacc = x[i];
#pragma unroll
                for (int j = 0; j < 32; j++) sacc = sacc - lv[j] * x[kb - 32 + j];
                x[i] = sacc;
            }
        }
        __syncthreads();
    }
#else
    __syncthreads();
    for (int kb = 0; kb < order; kb += 32) {
        const int nb = min(32, order - kb);
        if (warp == 0) {
            const bool mine = lane < nb;
            double xi = mine ? x[kb + lane] : 0.0;
            double lrow[32];
#pragma unroll
            for (int j = 0; j < 32; j++)
                lrow[j] = (mine && j < lane) ? __ldcg(L + (kb + lane) + (int64_t)(kb + j) * ldl) : 0.0;
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const double xj = __shfl_sync(FULL_MASK, xi, j);
                if (j < lane) xi = xi - lrow[j] * xj;
            }
            if (mine) x[kb + lane] = xi;
        }
        __syncthreads();
        for (int i = kb + nb + threadIdx.x; i < order; i += blockDim.x) {
            double lv[32];
#pragma unroll
            for (int j = 0; j < 32; j++) lv[j] = j < nb ? __ldcg(L + i + (int64_t)(kb + j) * ldl) : 0.0;
            double sacc = x[i];
#pragma unroll
            for (int j = 0; j < 32; j++)
                if (j < nb) sacc = sacc - lv[j] * x[kb + j];
            x[i] = sacc;
        }
        __syncthreads();
    }
#endif
}

// Givens rotation of H column j into R, update g; thread 0 does the
// sequential part from shared copies.  Returns |g[j+1]| to all threads.
__device__ __forceinline__ double givens_column(const Dev& d, int j, double* col, double* scs, double* ssn,
                                double* red) {
    const double* Hj = d.H + (int64_t)j * d.ldh;
    for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) col[i] = __ldcg(Hj + i);
    for (int i = threadIdx.x; i < j; i += blockDim.x) { scs[i] = __ldcg(d.cs + i); ssn[i] = __ldcg(d.sn + i); }
    __syncthreads();
    if (threadIdx.x == 0) {
        // the rotations chain through `carry`; operands are read 8 steps ahead (the stores
        // to col[] would otherwise order every shared load after the previous step)
        double carry = col[0];
        int i = 0;
        for (; i + 8 <= j; i += 8) {
            double bb[8], cc[8], ss[8];
#pragma unroll
            for (int k = 0; k < 8; k++) { bb[k] = col[i + k + 1]; cc[k] = scs[i + k]; ss[k] = ssn[i + k]; }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const double a = carry;
                col[i + k] = fma(cc[k], a, ss[k] * bb[k]);
                carry = fma(cc[k], bb[k], -ss[k] * a);
            }
        }
        for (; i < j; i++) {
            const double a = carry, b = col[i + 1];
            col[i] = fma(scs[i], a, ssn[i] * b);
            carry = fma(scs[i], b, -ssn[i] * a);
        }
        const double a = carry, b = col[j + 1];
        const double dd = hypot(a, b);
        double c = 1.0, s = 0.0;
        if (dd != 0.0) { c = a / dd; s = b / dd; }
        d.cs[j] = c;
        d.sn[j] = s;
        col[j] = dd;
        col[j + 1] = 0.0;
        const double gj = __ldcg(d.g + j);
        d.g[j + 1] = -s * gj;
        d.g[j] = c * gj;
        red[33] = fabs(-s * gj);
    }
    __syncthreads();
    double* Rj = d.R + (int64_t)j * d.ldh;
    for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) Rj[i] = col[i];
    const double res = red[33];
    __syncthreads();
    return res;
}

// The small step on the calling CTA (any blockDim that is a multiple of 32, <= 1024).  All
// global loads bypass L1 (ld.global.cg): the persistent cycle kernel runs this on one CTA
// while other CTAs of the same grid produce its inputs.  sm: small_smem(d.m) bytes, red: 40.
// publish = false (persistent kernel, worker CTAs other than 0): the Alg. 3 critical step is
// computed without any global write, and without the live status check, from the same
// reduced dots -- bitwise the coefficients CTA 0 publishes; loc (shared, >= p + 3 doubles)
// receives gamma, the update mode and beta (alpha stays in sm[0..p)).
__device__ __forceinline__ void small_body(const Dev& d, int stage, int gs, int p, int m, double* sm, double* red,
                           bool publish = true, double* loc = nullptr, bool r3_ready = false,
                           unsigned long long* tp = nullptr) {
    // tp (IGS_PC_PROF=1, persistent tail): timestamps of the SS_TAIL sub-steps
    auto tstamp = [&](int k) {
        if (tp && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            tp[k] = t;
        }
    };
    const int t0 = (int)__ldcg(d.scal + SC_T0);  // first global iteration of this cycle (graph-invariant)
    const int M = d.m;
    double* s_a = sm;               // [M+1]  r2 (Alg. 3) / a (Alg. 2)
    double* s_c = s_a + (M + 1);    // [M+2]  c (and d)
    double* s_x = s_c + (M + 2);    // [M+2]  r3 / r1
    double* s_col = s_x + (M + 2);  // [M+2]  Givens column
    double* s_cs = s_col + (M + 2); // [M+1]
    double* s_sn = s_cs + (M + 1);  // [M+1]
    double* s_t = s_sn + (M + 1);   // [M+1]  r2/gamma
    int* ist = d.istate;
    const int tid = threadIdx.x;

    if (stage == SS_PRIME_NORM) {  // rho = ||r||, v_0 = r / rho
        if (tid == 0) {
            const double s = __ldcg(d.dots);
            const double rho = sqrt(s);
            d.g[0] = rho;
            d.scal[SC_RHO] = rho;
            d.scal[SC_GAMMA] = rho;
            ist[ST_STATUS] = isfinite(rho) ? RUNNING : STOP_NONFINITE;
            ist[ST_PDONE] = 0;
            ist[ST_BASIS] = 0;
            ist[ST_MODE] = 1;
            ist[ST_MODE_IT] = 0;
            ist[ST_CRITBD] = -1;
            d.scal[SC_LCUM] = 0.0;
            if (t0 == 0) d.lnorm[0] = 0.0;
        }
        return;
    }
    if (stage == SS_PRIME_H) {  // H_11 = v_1^T A v_1, u = A v_1 - H_11 v_1 (reading R2)
        if (tid == 0) {
            if (*(volatile int*)(ist + ST_STATUS) != RUNNING) { ist[ST_MODE] = 0; return; }
            const double h = __ldcg(d.dots + 1);
            if (gs == 1) d.H[0] = h;
            else d.HP[0] = h;
            d.beta[0] = h;
            d.scal[SC_GAMMA] = 1.0;
            ist[ST_BASIS] = 1;
            ist[ST_MODE] = isfinite(h) ? 2 : 0;
            ist[ST_MODE_IT] = 0;
            if (!isfinite(h)) ist[ST_STATUS] = STOP_NONFINITE;
        }
        return;
    }
    if (stage == SS_LSQ) {  // y = R^{-1} g  (back substitution)
        const int pp = *(volatile int*)(ist + ST_PDONE);
        for (int i = tid; i < pp; i += blockDim.x) s_x[i] = __ldcg(d.g + i);
        for (int j = pp - 1; j >= 0; j--) {
            __syncthreads();
            if (tid == 0) s_x[j] = s_x[j] / __ldcg(d.R + j + (int64_t)j * d.ldh);
            __syncthreads();
            const double yj = s_x[j];
            for (int i = tid; i < j; i += blockDim.x) s_x[i] = s_x[i] - __ldcg(d.R + i + (int64_t)j * d.ldh) * yj;
        }
        __syncthreads();
        for (int i = tid; i < pp; i += blockDim.x) d.y[i] = s_x[i];
        return;
    }

    if (stage == SS_CRIT2 && *(volatile int*)(ist + ST_STATUS) != RUNNING) {
        if (tid == 0) ist[ST_MODE] = 0;  // the second update must not run either
        return;
    }
    if (publish && *(volatile int*)(ist + ST_STATUS) != RUNNING) return;

    if (stage == SS_CRIT2) {
        // Alg. 2 two-reduce, second Gauss-Seidel sweep: r2 = V_{p+1}^T u is in
        // dots2; r3 = (I + L_{p+1})^{-1} r2 (Step 15); H[:p+1, p] = r1 + r3 (Step 17);
        // alpha = r3 for w = u - V_{p+1} r3 (Step 16)
        if (*(volatile int*)(ist + ST_MODE_IT) != p || *(volatile int*)(ist + ST_MODE) != 3) {
            if (tid == 0) ist[ST_MODE] = 0;
            return;
        }
        for (int i = tid; i <= p; i += blockDim.x) s_x[i] = __ldcg(d.dots2 + i);
        trisolve_smem(p + 1, d.L, M, s_x);
        for (int i = tid; i <= p; i += blockDim.x) {
            d.H[i + (int64_t)p * d.ldh] = __ldcg(d.H + i + (int64_t)p * d.ldh) + s_x[i];
            d.alpha[i] = s_x[i];
        }
        __syncthreads();
        if (tid == 0) ist[ST_MODE] = 1;  // the second update writes w in place
        return;
    }
    if (stage == SS_MGS_NORM) {
        // MGS-GMRES: gamma = ||w|| after the j+1 projections of column
        // j = p-1; H[p, p-1] = gamma, Givens, status; v_p = w / gamma by the update kernel
        const int j = p - 1;
        const double s2 = __ldcg(d.dots);
        const double gamma = sqrt(s2);
        double h2 = 0.0;
        for (int i = tid; i <= j; i += blockDim.x) {
            const double h = __ldcg(d.H + i + (int64_t)j * d.ldh);
            h2 += h * h;
        }
        const double hn2 = block_sum(h2, red);
        const bool bd = !(gamma > kBreakdownC * kEps * sqrt(hn2 + gamma * gamma));
        if (tid == 0) d.H[p + (int64_t)j * d.ldh] = gamma;
        __syncthreads();
        const double res = givens_column(d, j, s_col, s_cs, s_sn, red);
        const double tol = __ldcg(d.scal + SC_TOL), nb = __ldcg(d.scal + SC_NB);
        const bool nonfinite = !isfinite(s2) || !isfinite(res) || !isfinite(hn2);
        const bool conv = tol > 0.0 && res <= tol * nb;
        if (tid == 0) {
            d.res_hist[t0 + p] = res / nb;
            ist[ST_PDONE] = p;
            ist[ST_MODE_IT] = p;
            d.scal[SC_GAMMA] = gamma;
            if (nonfinite) { ist[ST_STATUS] = STOP_NONFINITE; ist[ST_MODE] = 0; }
            else if (bd) { ist[ST_STATUS] = STOP_BREAKDOWN; ist[ST_MODE] = 0; ist[ST_BASIS] = p; }
            else {
                ist[ST_MODE] = 1;
                ist[ST_BASIS] = p + 1;
                if (conv || p == m) ist[ST_STATUS] = conv ? STOP_CONVERGED : STOP_END;
            }
        }
        return;
    }

    const double* dv = d.dots + (int64_t)p * d.dld;
    const bool drain = (p == m);
    const double s = __ldcg(dv + p);

    if (stage == SS_CRIT) {
        // ---------------- critical path of iteration p (feeds the fused update) ----------
        tstamp(0);
        for (int i = tid; i < p; i += blockDim.x) s_a[i] = __ldcg(dv + i);
        if (!drain) for (int i = tid; i <= p; i += blockDim.x) s_c[i] = __ldcg(dv + p + 1 + i);
        double gamma, lrow2 = 0.0;
        bool bd;
        if (gs == 2) {
            // Step 6: lagged norm gamma = sqrt(||u||^2 - ||r2||^2)
            double part = 0.0;
            for (int i = tid; i < p; i += blockDim.x) part += s_a[i] * s_a[i];
            const double nr2 = block_sum(part, red);
            const double t = s - nr2;
            gamma = t > 0.0 ? sqrt(t) : 0.0;
            lrow2 = nr2;
            bd = !(t > kBreakdownC * kEps * s);  // S:274 / reading R12 cancellation guard
            if (publish)
                for (int i = tid; i < p; i += blockDim.x) d.alpha[i] = s_a[i];  // Step 10 uses r2
        } else {
            // Alg. 2 Step 6: gamma = ||w_{k-1}|| (fused into the single reduction)
            gamma = sqrt(s);
            double h2 = 0.0;
            for (int i = tid; i < p; i += blockDim.x) {
                const double h = __ldcg(d.H + i + (int64_t)(p - 1) * d.ldh);
                h2 += h * h;
            }
            const double hn2 = block_sum(h2, red);
            bd = !(gamma > kBreakdownC * kEps * sqrt(hn2 + gamma * gamma));  // reading R12
            double pa = 0.0;
            for (int i = tid; i < p; i += blockDim.x) pa += s_a[i] * s_a[i];
            lrow2 = block_sum(pa, red);
        }
        if (!isfinite(gamma)) bd = true;
        if (loc && tid == 0) {
            loc[0] = gamma;
            loc[1] = bd ? 0.0 : (drain ? 1.0 : 3.0);  // update mode (as ST_MODE)
        }
        if (!publish) {
            __syncthreads();
            if (bd || drain) return;
        }
        if (publish && tid == 0) {  // ||L||_F of this cycle: row p of L is (r2 or a) / gamma
            double cum = __ldcg(d.scal + SC_LCUM);
            if (!drain && !bd) cum += lrow2 / (gamma * gamma);
            d.scal[SC_LCUM] = cum;
            d.lnorm[t0 + p] = sqrt(cum);
        }
        if (publish && tid == 0) {
            d.gam[p] = gamma;
            d.cbd[p] = bd ? 1.0 : 0.0;
            d.scal[SC_GAMMA] = gamma;
            ist[ST_CRITBD] = bd ? p : -1;
            ist[ST_MODE] = bd ? 0 : (drain ? 1 : 3);
            ist[ST_MODE_IT] = p;
            if (gs == 1) d.H[p + (int64_t)(p - 1) * d.ldh] = gamma;  // gamma_{k-1} = H_{k-1,k-2}
        }
        if (bd || drain) return;
        __syncthreads();
        if (gs == 2) {
            // Steps 7-9: c /= gamma ; d /= gamma^2 ; L[p, :p] = r2 / gamma  (reading R4)
            const double dd = s_c[p] / (gamma * gamma);
            double part = 0.0;
            for (int i = tid; i < p; i += blockDim.x) {
                const double ci = s_c[i] / gamma;
                const double li = s_a[i] / gamma;
                if (publish) {
                    d.L[p + (int64_t)i * M] = li;
                    d.beta[i] = ci;
                }
                if (loc) loc[2 + i] = ci;
                part += li * ci;
            }
            // Step 12 (Stephen's trick): r1 = [c ; d - L[p,:p] . c]
            const double acc = block_sum(part, red);
            if (tid == 0) {
                if (publish) d.beta[p] = dd - acc;
                if (loc) loc[2 + p] = dd - acc;
            }
            __syncthreads();
            if (publish) {
                double* r1row = d.r1h + (int64_t)p * (M + 2);  // copy for the tail (hp, Step 15)
                for (int i = tid; i <= p; i += blockDim.x) r1row[i] = __ldcg(d.beta + i);
            }
        } else {
            // Alg. 2 Steps 8-10: c /= gamma ; c[p] /= gamma ; L[p, :p] = a / gamma
            for (int i = tid; i <= p; i += blockDim.x) {
                double ci = s_c[i] / gamma;
                if (i == p) ci = ci / gamma;  // reading R5
                s_x[i] = ci;
            }
            for (int i = tid; i < p; i += blockDim.x) d.L[p + (int64_t)i * M] = s_a[i] / gamma;
            __threadfence_block();
            // Step 12: r1 = (I + L_{p+1})^{-1} c ; Step 17 (r3 = 0): H[:p+1, p] = r1
            tstamp(1);
            trisolve_smem(p + 1, d.L, M, s_x);
            tstamp(2);
            for (int i = tid; i <= p; i += blockDim.x) {
                d.beta[i] = s_x[i];
                d.H[i + (int64_t)p * d.ldh] = s_x[i];
            }
            __syncthreads();
            tstamp(3);
        }
        return;
    }

    // ---------------- SS_TAIL: Hessenberg column p-1, Givens, status, hp ------------------
    tstamp(0);
    const double tol = __ldcg(d.scal + SC_TOL), nb = __ldcg(d.scal + SC_NB);
    const double gamma = __ldcg(d.gam + p);
    bool bd = __ldcg(d.cbd + p) != 0.0;
    double hn2 = 0.0;
    if (gs == 2) {
        // Step 5: r3 = (I + L_p)^{-1} r2 ; Step 14: H[:p, p-1] = hp + r3, H[p, p-1] = gamma (R3)
        if (r3_ready) {  // computed ahead by the persistent kernel's forward-substitution CTA
            for (int i = tid; i < p; i += blockDim.x) s_x[i] = __ldcg(d.r3h + (int64_t)p * (M + 2) + i);
        } else {
            for (int i = tid; i < p; i += blockDim.x) s_x[i] = __ldcg(dv + i);
            trisolve_smem(p, d.L, M, s_x);
        }
        double h2 = 0.0;
        for (int i = tid; i < p; i += blockDim.x) {
            const double h = __ldcg(d.HP + i + (int64_t)(p - 1) * d.ldh) + s_x[i];
            d.H[i + (int64_t)(p - 1) * d.ldh] = h;
            h2 += h * h;
        }
        hn2 = block_sum(h2, red);
        if (!(gamma > kBreakdownC * kEps * sqrt(hn2 + gamma * gamma))) bd = true;  // reading R12
        if (tid == 0) d.H[p + (int64_t)(p - 1) * d.ldh] = gamma;
        __syncthreads();
    }
    tstamp(1);
    const double res = givens_column(d, p - 1, s_col, s_cs, s_sn, red);
    tstamp(2);
    const bool nonfinite = !isfinite(s) || !isfinite(res) || !isfinite(hn2) || !isfinite(gamma);
    const bool conv = tol > 0.0 && res <= tol * nb;
    if (tid == 0) {
        d.res_hist[t0 + p] = res / nb;
        ist[ST_PDONE] = p;
        if (nonfinite) ist[ST_STATUS] = STOP_NONFINITE;
        else if (bd) { ist[ST_STATUS] = STOP_BREAKDOWN; ist[ST_BASIS] = p; }
        else {
            ist[ST_BASIS] = p + 1;
            if (conv || drain) ist[ST_STATUS] = conv ? STOP_CONVERGED : STOP_END;
        }
    }
    if (gs == 1 || nonfinite || bd || conv || drain) return;
    // Step 15, derived (reading R1): hp[:p+1, p] = r1 - H[:p+1, :p] (r2 / gamma); H is upper
    // Hessenberg, so row i only meets columns j >= i-1 (the skipped terms are exact zeros)
    // Work items = (32-row block, chunk of T consecutive columns): a warp's lanes are the 32
    // rows (H is column-major: one coalesced 256-byte load per column), 16 columns in flight
    // per lane; row block rb meets columns j >= 32 rb - 1 only, and inside it the entries
    // below the subdiagonal are skipped (exact zeros).  T balances the items over the warps;
    // partials are combined per row in column order.
    tstamp(3);
    for (int j = tid; j < p; j += blockDim.x) s_t[j] = __ldcg(d.L + p + (int64_t)j * M);
    const int rows = p + 1;
    double* s_part = s_col;  // s_col | s_cs | s_sn: 3M + 4 doubles, free after Givens
    const int nrb = (rows + 31) / 32, nwarps = (int)(blockDim.x >> 5);
    auto rb_j0 = [&](int rb) { return rb > 0 ? 32 * rb - 1 : 0; };
    int sumlen = 0;
    for (int rb = 0; rb < nrb; rb++) sumlen += p - rb_j0(rb);
    int T = max(16, (sumlen + nwarps - 1) / nwarps);
    auto items = [&](int tt) {
        int c = 0;
        for (int rb = 0; rb < nrb; rb++) c += (p - rb_j0(rb) + tt - 1) / tt;
        return c;
    };
    while (items(T) * 32 > 3 * M + 4 && T < p) T *= 2;
    if (T > p) T = p;
    const int nit = items(T);
    __syncthreads();
    if (nit * 32 > 3 * M + 4) {  // tiny M (< 14): one thread per row, columns in order
        for (int i = tid; i < rows; i += blockDim.x) {
            double sacc = 0.0;
            for (int j = i > 0 ? i - 1 : 0; j < p; j++) sacc += __ldcg(d.H + i + (int64_t)j * d.ldh) * s_t[j];
            d.HP[i + (int64_t)p * d.ldh] = __ldcg(d.r1h + (int64_t)p * (M + 2) + i) - sacc;
        }
        __syncthreads();
        tstamp(4);
        __syncthreads();
        tstamp(5);
        return;
    }
    for (int it = (int)(threadIdx.x >> 5); it < nit; it += nwarps) {
        int rb = 0, base = 0;
        for (;; rb++) {
            const int c = (p - rb_j0(rb) + T - 1) / T;
            if (it < base + c) break;
            base += c;
        }
        const int i = 32 * rb + (tid & 31);
        int j = rb_j0(rb) + (it - base) * T;
        const int e = min(j + T, p);
        double sacc = 0.0;
        for (; j < e; j += 16) {
            double hv[16];
#pragma unroll
            for (int c = 0; c < 16; c++)
                hv[c] = (j + c < e && i < rows && i <= j + c + 1) ? __ldcg(d.H + i + (int64_t)(j + c) * d.ldh) : 0.0;
#pragma unroll
            for (int c = 0; c < 16; c++)
                if (j + c < e && i <= j + c + 1) sacc += hv[c] * s_t[j + c];
        }
        s_part[it * 32 + (tid & 31)] = sacc;
    }
    __syncthreads();
    tstamp(4);
    for (int i = tid; i < rows; i += blockDim.x) {
        const int rb = i >> 5;
        int k0 = 0;
        for (int r = 0; r < rb; r++) k0 += (p - rb_j0(r) + T - 1) / T;
        const int k1 = k0 + (p - rb_j0(rb) + T - 1) / T;
        double sacc = 0.0;
        for (int k = k0; k < k1; k++) sacc += s_part[k * 32 + (i & 31)];
        d.HP[i + (int64_t)p * d.ldh] = __ldcg(d.r1h + (int64_t)p * (M + 2) + i) - sacc;
    }
    __syncthreads();
    tstamp(5);
}

__global__ void __launch_bounds__(SS_THREADS)
    small_kernel(Dev d, int stage, int gs, int p, int m, int t0_unused) {
    extern __shared__ double sm[];
    __shared__ double red[40];
    small_body(d, stage, gs, p, m, sm, red);
}

static size_t small_smem(int M) { return (size_t)(7 * (M + 2)) * sizeof(double); }

void launch_small(const Dev& d, int stage, int gs, int p, int m, int t0, cudaStream_t s) {
    const size_t smem = small_smem(d.m);
    if (smem > 48 * 1024) cudaFuncSetAttribute(small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    small_kernel<<<1, SS_THREADS, smem, s>>>(d, stage, gs, p, m, t0);
}

// ------------------------------------------------------------------------------------
// Algorithm 1 small steps, one CTA (igs_qr).  Workspace layout in QrDev.
//   QR_S0     R_11 = ||a_1||                                  (Step 1)
//   QR_S1     R_12 = q_1^T a_2                                (Step 2)
//   QR_CRIT   column k >= 2: gamma_{k-1} = ||w_{k-1}|| = R_{k-1,k-1} (Step 5), L row (Step 8),
//             r0 with only its last entry divided by gamma (Step 7, reading R22),
//             r1 = (I + L)^{-1} r0 (Step 9), R[:k, k] = r1;  drain (k = m): gamma only
//   QR_CRIT2  r3 = (I + L)^{-1} r2 (Step 12), R[:k, k] += r3 (Step 14), alpha = r3 (Step 13)
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(SS_THREADS) qr_small_kernel(QrDev q, int stage, int k, int m) {
    extern __shared__ double qs[];
    const int tid = threadIdx.x;
    double* R = q.R;
    if (stage == QR_S0) {
        if (tid == 0) { const double g = sqrt(q.dots[0]); R[0] = g; q.scal[0] = g; q.scal[1] = 1.0; }
        return;
    }
    if (stage == QR_S1) {
        if (tid == 0) { const double h = q.dots[1]; R[(int64_t)m] = h; q.beta[0] = h; }
        return;
    }
    if (stage == QR_CRIT) {
        const int p = k - 1;                   // normalised columns before w_{k-1}
        const double* dv = q.dots;             // [Q_p^T w (p), w.w, Q_p^T a_k (p), w.a_k]
        const double gamma = sqrt(dv[p]);
        if (tid == 0) { R[p + (int64_t)p * m] = gamma; q.scal[0] = gamma; }
        if (k == m) return;                    // drain: normalise the last column only
        for (int i = tid; i < p; i += blockDim.x) {
            q.L[p + (int64_t)i * m] = dv[i] / gamma;    // Step 8
            qs[i] = dv[p + 1 + i];                       // Step 7: r0 entries of q_0..q_{p-1}
        }
        if (tid == 0) qs[p] = dv[2 * p + 1] / gamma;     // ... and of the new q_p = w / gamma
        trisolve_smem(k, q.L, m, qs);                    // Step 9 (order k = p + 1)
        for (int i = tid; i < k; i += blockDim.x) {
            q.beta[i] = qs[i];
            R[i + (int64_t)k * m] = qs[i];               // Step 14 (first part)
        }
        return;
    }
    if (stage == QR_CRIT2) {
        for (int i = tid; i < k; i += blockDim.x) qs[i] = q.dots2[i];
        trisolve_smem(k, q.L, m, qs);                    // Step 12
        for (int i = tid; i < k; i += blockDim.x) {
            R[i + (int64_t)k * m] = R[i + (int64_t)k * m] + qs[i];   // Step 14: r1 + r3
            q.alpha[i] = qs[i];                                      // Step 13 coefficients
        }
        return;
    }
}

void launch_qr_small(const QrDev& q, int stage, int k, int m, cudaStream_t s) {
    const size_t smem = (size_t)(m + 2) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(qr_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qr_small_kernel<<<1, SS_THREADS, smem, s>>>(q, stage, k, m);
}

__global__ void __launch_bounds__(SS_THREADS)
    trisolve_kernel(int order, const double* L, int ldl, const double* b, double* x) {
    extern __shared__ double sx[];
    for (int i = threadIdx.x; i < order; i += blockDim.x) sx[i] = b[i];
    trisolve_smem(order, L, ldl, sx);
    for (int i = threadIdx.x; i < order; i += blockDim.x) x[i] = sx[i];
}

void launch_trisolve(int order, const double* L, int ldl, const double* b, double* x,
                     cudaStream_t s) {
    const size_t smem = (size_t)(order + 1) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(trisolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    trisolve_kernel<<<1, SS_THREADS, smem, s>>>(order, L, ldl, b, x);
}

// ------------------------------------------------------------------------------------
// LOO diagnostic: G = V^T V (tiled, deterministic), ||I - G||_F
// Each thread sums 4096-row pieces with FMAs and adds the pieces into a compensated
// (Neumaier) running sum; the splits are combined the same way.  A plain running sum over a
// split of 2.1M rows (c5: 134M rows / 64) drifted by ~1e-12 per entry -- LOO 6.9e-11 against
// ~1e-12 from the same basis -- i.e. the diagnostic measured its own rounding.
// ------------------------------------------------------------------------------------
constexpr int GR_T = 32, GR_R = 64, GR_PIECE = 64;  // GR_PIECE tiles of GR_R rows per piece

__device__ __forceinline__ void neumaier_add(double& s, double& comp, double x) {
    const double t = s + x;
    comp += (fabs(s) >= fabs(x)) ? (s - t) + x : (x - t) + s;
    s = t;
}

__global__ void __launch_bounds__(256)
    gram_kernel(int64_t n, int c, const double* __restrict__ V, int64_t ld,
                double* __restrict__ part, int ntile) {
    __shared__ double A[GR_T][GR_R + 1];
    __shared__ double B[GR_T][GR_R + 1];
    // tile pair (ti <= tj) from blockIdx.x
    int idx = blockIdx.x, ti = 0;
    while (idx >= ntile - ti) { idx -= ntile - ti; ti++; }
    const int tj = ti + idx;
    const int split = blockIdx.y, splits = gridDim.y;
    const int64_t chunk = (n + splits - 1) / splits;
    const int64_t rbeg = (int64_t)split * chunk;
    const int64_t rend = rbeg + chunk < n ? rbeg + chunk : n;
    const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    double sum[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, comp[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    int pieces = 0;
    for (int64_t r0 = rbeg; r0 < rend; r0 += GR_R) {
        for (int e = threadIdx.x; e < GR_T * GR_R; e += 256) {
            const int cc = e / GR_R, rr = e % GR_R;
            const int64_t row = r0 + rr;
            const int ca = ti * GR_T + cc, cb = tj * GR_T + cc;
            A[cc][rr] = (row < rend && ca < c) ? V[(int64_t)ca * ld + row] : 0.0;
            B[cc][rr] = (row < rend && cb < c) ? V[(int64_t)cb * ld + row] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = 0; rr < GR_R; rr++) {
            const double a0 = A[2 * ty][rr], a1 = A[2 * ty + 1][rr];
            const double b0 = B[2 * tx][rr], b1 = B[2 * tx + 1][rr];
            acc[0][0] = fma(a0, b0, acc[0][0]);
            acc[0][1] = fma(a0, b1, acc[0][1]);
            acc[1][0] = fma(a1, b0, acc[1][0]);
            acc[1][1] = fma(a1, b1, acc[1][1]);
        }
        __syncthreads();
        if (++pieces == GR_PIECE) {
            pieces = 0;
            for (int a = 0; a < 2; a++)
                for (int b = 0; b < 2; b++) { neumaier_add(sum[a][b], comp[a][b], acc[a][b]); acc[a][b] = 0.0; }
        }
    }
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++) {
            neumaier_add(sum[a][b], comp[a][b], acc[a][b]);
            const int i = ti * GR_T + 2 * ty + a, j = tj * GR_T + 2 * tx + b;
            if (i < c && j < c) part[((int64_t)split * c + i) * c + j] = sum[a][b] + comp[a][b];
        }
}

__global__ void gram_reduce_kernel(int c, int splits, const double* __restrict__ part, double* G) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)c * c) return;
    const int i = (int)(e / c), j = (int)(e % c);
    const int a = i < j ? i : j, b = i < j ? j : i;  // computed entries live in the upper part
    double s = 0.0, comp = 0.0;
    for (int k = 0; k < splits; k++) neumaier_add(s, comp, part[((int64_t)k * c + a) * c + b]);
    G[e] = s + comp;
}

void launch_gram(int64_t n, int c, const double* V, int64_t ld, double* part, int splits,
                 double* G, cudaStream_t s) {
    const int ntile = (c + GR_T - 1) / GR_T;
    dim3 grid(ntile * (ntile + 1) / 2, splits);
    gram_kernel<<<grid, 256, 0, s>>>(n, c, V, ld, part, ntile);
    const int64_t tot = (int64_t)c * c;
    gram_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c, splits, part, G);
}

// out[0] = ||I - G||_F; out[1] = ||tril(G, -1)||_F, the paper's L_k of the
// computed basis (strictly lower part of V^T V; dep^2(I + L_k) = ||L_k||_F^2,
// P:1216-1223).  gram_reduce_kernel mirrors one computed triangle, so G is exactly
// symmetric and either triangle gives the same norm.
__global__ void loo_norm_kernel(int c, const double* __restrict__ G, double* out) {
    __shared__ double red[40];
    double part = 0.0, low = 0.0;
    for (int64_t e = threadIdx.x; e < (int64_t)c * c; e += blockDim.x) {
        const int i = (int)(e / c), j = (int)(e % c);
        const double d = (i == j ? 1.0 : 0.0) - G[e];
        part += d * d;
        if (j > i) low += G[e] * G[e];
    }
    const double s = block_sum(part, red);
    __syncthreads();
    const double l = block_sum(low, red);
    if (threadIdx.x == 0) { out[0] = sqrt(s); out[1] = sqrt(l); }
}

void launch_loo_norm(int c, const double* G, double* out, cudaStream_t s) {
    loo_norm_kernel<<<1, 256, 0, s>>>(c, G, out);
}

// ------------------------------------------------------------------------------------
__global__ void mgs_axpy_kernel(int64_t n, const double* __restrict__ v, double* __restrict__ z,
                                const double* __restrict__ hsrc, double* Hdst, const int* istate) {
    if (!running(istate)) return;
    const double h = *hsrc;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *Hdst = h;
    if (i < n) z[i] = z[i] - h * v[i];
}

void launch_mgs_axpy(int64_t n, const double* v, double* z, const double* hsrc, double* Hdst,
                     const int* istate, cudaStream_t s) {
    mgs_axpy_kernel<<<(unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1), 256, 0, s>>>(n, v, z, hsrc, Hdst, istate);
}

// MGS projection i of column j fused with the inner product that follows it (the
// modified Gram-Schmidt loop taken in its own order):  with h = v_i . w from the previous
// reduction,  H[i,j] = h;  w <- w - h v_i;  then  out = v_{i+1} . w  (or w . w after the last
// projection).  One pass over v_i, w, v_{i+1} instead of a dot pass and an axpy pass; the
// FMA and every per-element operation are those of the two-kernel sequence.  AXPY = false:
// the first dot of a column (no projection yet).  Each thread owns 4 rows of a 1024-row
// chunk (two 16-byte loads per vector), grid-stride; deterministic two-stage sum: per-CTA
// partials in a fixed tree, the last CTA to arrive sums them in CTA order with a fixed
// per-thread split (+ across ranks over NVLink when xc != nullptr).
constexpr int MS_THREADS = 256;
constexpr int MS_CHUNK = 4 * MS_THREADS;

template <bool AXPY, bool NORM>
__global__ void __launch_bounds__(MS_THREADS)
    mgs_step_kernel(int64_t n, const double* __restrict__ v, double* __restrict__ z,
                    const double* __restrict__ vn, const double* hsrc, double* Hdst,
                    double* __restrict__ part, double* out, unsigned* counter, const int* istate,
                    const XchgDev* xc) {
    const bool live = running(istate);  // stopped: with the exchange, join it without work
    if (!live && !xc) return;
    __shared__ double red[40];
    __shared__ bool s_last;
    const double h = AXPY && live ? __ldcg(hsrc) : 0.0;
    if (AXPY && live && blockIdx.x == 0 && threadIdx.x == 0) *Hdst = h;
    double acc = 0.0;
    const int64_t nfull = live ? n / MS_CHUNK : 0;
    for (int64_t c = blockIdx.x; c < nfull; c += gridDim.x) {
        const int64_t r0 = c * MS_CHUNK + 2 * threadIdx.x, r1 = r0 + 2 * MS_THREADS;
        double2 w0 = __ldcg(reinterpret_cast<const double2*>(z + r0));
        double2 w1 = __ldcg(reinterpret_cast<const double2*>(z + r1));
        double2 q0, q1;
        if (!NORM) {
            q0 = __ldg(reinterpret_cast<const double2*>(vn + r0));
            q1 = __ldg(reinterpret_cast<const double2*>(vn + r1));
        }
        if (AXPY) {
            const double2 a0 = __ldg(reinterpret_cast<const double2*>(v + r0));
            const double2 a1 = __ldg(reinterpret_cast<const double2*>(v + r1));
            w0.x = w0.x - h * a0.x;
            w0.y = w0.y - h * a0.y;
            w1.x = w1.x - h * a1.x;
            w1.y = w1.y - h * a1.y;
            *reinterpret_cast<double2*>(z + r0) = w0;
            *reinterpret_cast<double2*>(z + r1) = w1;
        }
        if (NORM) q0 = w0, q1 = w1;
        acc = fma(q0.x, w0.x, acc);
        acc = fma(q0.y, w0.y, acc);
        acc = fma(q1.x, w1.x, acc);
        acc = fma(q1.y, w1.y, acc);
    }
    // ragged tail (< MS_CHUNK rows): the last CTA of the chunk loop's next round, one row per thread
    if (live && (int64_t)blockIdx.x == nfull % gridDim.x) {
        for (int64_t r = nfull * MS_CHUNK + threadIdx.x; r < n; r += MS_THREADS) {
            double w = z[r];
            if (AXPY) {
                w = w - h * v[r];
                z[r] = w;
            }
            acc = fma(NORM ? w : vn[r], w, acc);
        }
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double t = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += MS_THREADS) t += __ldcg(part + b);
    t = block_sum(t, red);
    if (xc) {
        if (threadIdx.x == 0) part[gridDim.x] = t;
        __threadfence();
        __syncthreads();
        final_reduce_xchg(part + gridDim.x, 1, 1, out, *xc);
    } else if (threadIdx.x == 0) {
        *out = t;
    }
    if (threadIdx.x == 0) { *counter = 0u; counter[1] += live ? 1u : 0u; }
}

int mgs_step_grid(int64_t n, int num_sms) {
    const int64_t chunks = (n + MS_CHUNK - 1) / MS_CHUNK;
    int64_t g = (int64_t)num_sms * 4;
    if (g > chunks) g = chunks;
    return (int)(g < 1 ? 1 : g);
}

void launch_mgs_step(int64_t n, const double* v, double* z, const double* vn, const double* hsrc,
                     double* Hdst, double* part, double* out, unsigned* counter, int grid,
                     const int* istate, const XchgDev* xc, cudaStream_t s) {
    if (v && vn)
        mgs_step_kernel<true, false><<<grid, MS_THREADS, 0, s>>>(n, v, z, vn, hsrc, Hdst, part, out, counter, istate, xc);
    else if (v)
        mgs_step_kernel<true, true><<<grid, MS_THREADS, 0, s>>>(n, v, z, vn, hsrc, Hdst, part, out, counter, istate, xc);
    else
        mgs_step_kernel<false, false><<<grid, MS_THREADS, 0, s>>>(n, v, z, vn, hsrc, Hdst, part, out, counter, istate, xc);
}

__global__ void pack_kernel(int64_t cnt, const int64_t* __restrict__ idx,
                            const double* __restrict__ x, double* __restrict__ buf,
                            const int* istate) {
    if (!running(istate)) return;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) buf[i] = x[idx[i]];
}

void launch_pack(int64_t cnt, const int64_t* idx, const double* x, double* buf, const int* istate,
                 cudaStream_t s) {
    if (cnt <= 0) return;
    pack_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(cnt, idx, x, buf, istate);
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// out[i] = sum over q = 0..G-1 of stage[q][i], in member order (igs_virtual_solve's
// emulated allreduce; the same order on every member)
__global__ void rank_sum_kernel(const double* const* __restrict__ stage, int G, int64_t count,
                                double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    double s = 0.0;
    for (int q = 0; q < G; q++) s += stage[q][i];
    out[i] = s;
}

void launch_rank_sum(const double* const* stage, int G, int64_t count, double* out, cudaStream_t s) {
    if (count <= 0) return;
    rank_sum_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(stage, G, count, out);
}

void launch_fill(double* p, int64_t n, double v, cudaStream_t s) {
    if (n <= 0) return;
    fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, v);
}


// ------------------------------------------------------------------------------------
// Persistent cycle kernel ("a persistent cooperative kernel for tiny
// n").  Iterations p = 1..m of one cycle in ONE cooperative launch, for small single-GPU
// problems where the 4-5 dependent launches per iteration, not bytes, set the time.  Same
// algebra as the per-kernel path (Alg. 3 for gs = 2, Alg. 2 one sweep for gs = 1).
// Worker CTAs 0..W-1 run the phases of iteration p separated by grid barriers:
//   A  z = A u                  lpr lanes per row                             (Step 4)
//   B  the 2(p+1) dots          CTA b owns a contiguous range of the columns c of
//                               [V_p, u] and forms V_c.u and V_c.z over all n rows, so
//                               no cross-CTA partial sums exist (deterministic) (Step 4)
//   C  critical small step      CTA 0: small_body(SS_CRIT), or the stop decision
//   D  fused update             32-row tiles; the warps of a CTA split tiles x columns
// The last CTA (W = G-1 when G > 1) runs the tail small step (r3, H column, Givens,
// residual, status, hp; SS_TAIL) of iteration p as soon as CRIT(p) is published, trailing
// the workers by at most PC_LAG iterations (CRIT(p) waits for TAIL(p - PC_LAG)); a stop the
// tail decides is acted on at the next C phase.  Every load of data written inside the
// launch is ld.global.cg: L1 is not coherent across SMs.
// flags (zeroed before launch): [0] barrier count, [1] last p whose CRIT ran, [2] p at
// which CTA 0 stopped (0 = running), [3] last p whose TAIL ran, [4] first p whose TAIL
// left the status not RUNNING, [5] last p whose dots are final, [6] last p whose r3 is
// computed (forward-substitution CTA, Alg. 3; [7]: the second such CTA's, odd p).
// ------------------------------------------------------------------------------------
constexpr int PC_THREADS = 512;
constexpr int PC_WARPS = PC_THREADS / 32;
constexpr int PC_CB = 8;   // dot columns per register block
#ifndef PC_LAG_ITERS
#define PC_LAG_ITERS 2
#endif
constexpr int PC_LAG = PC_LAG_ITERS;  // iterations the tail CTA may trail the critical step
#ifndef PC_XS_UNROLL
#define PC_XS_UNROLL 8       // staged-u CSR phase: loads in flight per lane
#endif
#ifndef PC_XS_PRED
#define PC_XS_PRED 0         // 1: predicated last round instead of a one-by-one remainder
#endif
#ifndef PC_ROW_INTERLEAVE
#define PC_ROW_INTERLEAVE 1  // row groups dealt round-robin over CTAs first (0: CTA-contiguous)
#endif

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        epoch += 1u;
        const unsigned target = epoch * nblocks;
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) {
        }
    }
    __syncthreads();
}

template <typename IT, typename PT>
__global__ void __launch_bounds__(PC_THREADS, 1)
    pcycle_kernel(Dev d, int64_t n, int m, int gs, const PT* __restrict__ rowptr,
                  const IT* __restrict__ col, const double* __restrict__ val, int lpr, double* V,
                  int64_t ld, double* z, unsigned* flags, unsigned* counter, unsigned long long* prof,
                  double* part, SellDev<IT> sell, int xs, int ntri, int ares) {
    extern __shared__ double sm[];
    __shared__ double red[40];
    __shared__ int s_go;
    const int M = d.m;
    auto stamp = [&](int p, int k) {  // phase timestamps (IGS_PC_PROF=1), CTA 0 / tail CTA
        if (prof && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prof[(int64_t)p * 8 + k] = t;
        }
    };
    double* s_small = sm;                        // small_smem(M)
    double* s_coef = sm + 7 * (M + 2);           // alpha [M+1] | beta [M+1]
    double* s_red = s_coef + 2 * (M + 1);        // [PC_WARPS][2 * PC_CB] (B) / [2][PC_WARPS][32] (D)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const bool split = G > 1;
    // Alg. 3 with >= 3 CTAs: CTA G-2 computes the Step 5 forward substitution r3 of iteration
    // p as soon as its dots and L row p-1 are final, ahead of the tail (which then only does
    // H, Givens and the Step 15 GEMV)
    // ntri = 2: two such CTAs take alternate iterations (a forward substitution of order p
    // per iteration is the slowest serial chain at large m); the critical-step publishes
    // stay in iteration order (CTA t publishes CRIT(p) only after CRIT(p-1))
    const int nt = (gs == 2 && G >= 3) ? max(1, min(ntri, G - 2)) : 0;
    const bool tri = nt > 0;
    const int W = split ? G - 1 - nt : 1;  // worker CTAs
    const volatile int* vist = d.istate;

    if (tri && b >= G - 1 - nt && b <= G - 2) {
        const int ti = G - 2 - b;  // this CTA takes the iterations p with p % nt == ti
        // ---------------- forward-substitution CTA ---------------------------------------
        // also the published copy of the critical step (L row, r1, gamma, lnorm, mode
        // words), so no worker pays for those global writes; the workers compute the same
        // coefficients locally.  L row p-1 (for this iteration's solve) is its own earlier
        // output.
        double* s_x = s_small + (M + 1) + (M + 2);  // small_body's s_x slot
        for (int p = ti > 0 ? ti : nt; p <= m; p += nt) {
            if (tid == 0) {
                int go = 0;
                while (true) {  // dots of p final and CRIT(p-1) published
                    if (ld_acquire_u32(flags + 5) >= (unsigned)p && ld_acquire_u32(flags + 1) + 1u >= (unsigned)p) { go = 1; break; }
                    if (ld_acquire_u32(flags + 2) != 0u) {
                        go = ld_acquire_u32(flags + 5) >= (unsigned)p && ld_acquire_u32(flags + 1) + 1u >= (unsigned)p;
                        break;
                    }
                }
                s_go = go;
            }
            __syncthreads();
            if (!s_go) break;
            small_body(d, SS_CRIT, gs, p, m, s_small, red);
            __syncthreads();
            if (tid == 0) { __threadfence(); st_release_u32(flags + 1, (unsigned)p); }
            const double* dv = d.dots + (int64_t)p * d.dld;
            for (int i = tid; i < p; i += PC_THREADS) s_x[i] = __ldcg(dv + i);
            trisolve_smem(p, d.L, M, s_x);
            for (int i = tid; i < p; i += PC_THREADS) d.r3h[(int64_t)p * (M + 2) + i] = s_x[i];
            __syncthreads();
            if (tid == 0) { __threadfence(); st_release_u32(flags + 6 + ti, (unsigned)p); }
        }
        return;
    }

    if (split && b == G - 1) {
        // ---------------- tail CTA ---------------------------------------------------------
        // Alg. 3 without a forward-substitution CTA: this CTA runs the published copy of the
        // critical step (see above) as soon as the dots of p are final
        const bool own_crit = gs == 2 && !tri;
        for (int p = 1; p <= m; p++) {
            if (own_crit) {
                if (tid == 0) {
                    int go = 0;
                    while (true) {
                        if (ld_acquire_u32(flags + 5) >= (unsigned)p) { go = 1; break; }
                        if (ld_acquire_u32(flags + 2) != 0u) { go = ld_acquire_u32(flags + 5) >= (unsigned)p; break; }
                    }
                    s_go = go;
                }
                __syncthreads();
                if (!s_go) break;
                small_body(d, SS_CRIT, gs, p, m, s_small, red);
                __syncthreads();
                if (tid == 0) { __threadfence(); st_release_u32(flags + 1, (unsigned)p); }
            }
            if (tid == 0) {
                const unsigned* r3f = flags + 6 + (tri ? p % nt : 0);  // r3 of p: its CTA's word
                int go = 0;
                while (true) {
                    if (ld_acquire_u32(flags + 1) >= (unsigned)p && (!tri || ld_acquire_u32(r3f) >= (unsigned)p)) { go = 1; break; }
                    if (ld_acquire_u32(flags + 2) != 0u) {  // stopped: CRIT(p) may still have run
                        go = ld_acquire_u32(flags + 1) >= (unsigned)p;
                        if (go && tri)  // its r3 follows: the dots of p were final before CRIT(p)
                            while (ld_acquire_u32(r3f) < (unsigned)p) {
                            }
                        break;
                    }
                }
                s_go = go;
                if (go && vist[ST_STATUS] == RUNNING) counter[1] += 1u;  // reductions executed
            }
            __syncthreads();
            if (!s_go) break;
            stamp(p, 6);
            small_body(d, SS_TAIL, gs, p, m, s_small, red, true, nullptr, /*r3_ready=*/tri,
                       prof ? prof + (int64_t)(m + 2) * 8 + (int64_t)p * 8 : nullptr);
            stamp(p, 7);
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                // first iteration at which the status left RUNNING (the workers' stop rule)
                if (vist[ST_STATUS] != RUNNING && ld_acquire_u32(flags + 4) == 0u) st_release_u32(flags + 4, (unsigned)p);
                st_release_u32(flags + 3, (unsigned)p);
            }
        }
        return;
    }

    // ---------------- worker CTAs ----------------------------------------------------------
    unsigned epoch = 0;
    if (vist[ST_STATUS] != RUNNING) {  // stopped by the cycle priming (final at launch: uniform)
        if (b == 0 && tid == 0) { __threadfence(); st_release_u32(flags + 2, 1u); }
        return;
    }
    // ares > 0 (with xs, 32 lanes per row): the CTA's rows of A stay in shared memory for the
    // whole cycle -- the row assignment of phase A is static (warp w of CTA b: rows w W + b,
    // + 16 W, ...), so warp w copies its rows' values and (16-bit) columns once, in CSR order,
    // behind the staged u; per iteration phase A then reads A from shared memory instead of
    // 4 dependent L2 round trips per long row (c2: 24 MB of CSR = 162 KB per SM).  Same
    // entries in the same order per lane: bitwise the plain phase.
    //   layout after s_xs[n]: values [ares] | columns uint16 [ares] | row lengths int [PC_WARPS K]
    double* s_av = s_red + 2 * PC_WARPS * 32 + n;
    unsigned short* s_ac = reinterpret_cast<unsigned short*>(s_av + ares);
    int* s_rl = reinterpret_cast<int*>(s_ac + ((ares + 3) & ~3));
    __shared__ int s_woff[PC_WARPS + 1];
    const int rstep = W * PC_WARPS;  // rows between two rows of the same warp
    if (ares > 0) {
        if (tid < PC_WARPS) {
            int tot = 0, k = 0;
            for (int64_t r = (int64_t)tid * W + b; r < n; r += rstep, k++) {
                const int len = (int)(__ldg(rowptr + r + 1) - __ldg(rowptr + r));
                s_rl[k * PC_WARPS + tid] = len;
                tot += len;
            }
            s_woff[tid + 1] = tot;
        }
        __syncthreads();
        if (tid == 0) {
            s_woff[0] = 0;
            for (int w = 0; w < PC_WARPS; w++) s_woff[w + 1] += s_woff[w];
        }
        __syncthreads();
        int o = s_woff[warp];
        for (int64_t r = (int64_t)warp * W + b; r < n; r += rstep) {
            const int64_t q0 = (int64_t)__ldg(rowptr + r), q1 = (int64_t)__ldg(rowptr + r + 1);
            for (int64_t q = q0 + lane; q < q1; q += 32) {
                s_av[o + (int)(q - q0)] = __ldg(val + q);
                s_ac[o + (int)(q - q0)] = (unsigned short)__ldg(col + q);
            }
            o += (int)(q1 - q0);
        }
        __syncthreads();
    }
    for (int p = 1; p <= m; p++) {
        const bool drain = (p == m);
        const double* u = V + (int64_t)p * ld;
        if (b == 0) stamp(p, 0);
        // ---- A: z = A u (Step 4) ---------------------------------------------------------
        if (!drain && sell.ptr) {
            // SELL-32 copy (short rows): one thread per row, whole warps per slice (sell_row
            // shuffles), left-to-right separate multiply and add (bitwise the oracle's row loop)
            for (int64_t r = (int64_t)b * PC_THREADS + tid; (r & ~(int64_t)31) < n; r += (int64_t)W * PC_THREADS) {
                double sum;
                if (sell_row<IT, false, true, SELL_MIXED>(sell, r, r < n, u, nullptr, n, sum)) z[r] = sum;
            }
            grid_barrier(flags, W, epoch);
        } else if (!drain) {
            const int groups = 32 / lpr, sub = lane / lpr, sl = lane % lpr;
            const int64_t stride = (int64_t)W * PC_WARPS * groups;
            // xs (long rows, n <= PC_XS_MAX): u staged in shared memory first, so the gathers
            // leave the per-row dependency chain (same FMA sequence per lane: bitwise equal)
            double* s_xs = s_red + 2 * PC_WARPS * 32;
            if (xs && (int64_t)b * groups < n) {
                for (int64_t i = tid; i < n; i += PC_THREADS) s_xs[i] = __ldcg(u + i);
                __syncthreads();
            }
            if (ares > 0) {  // A resident in shared memory (lpr = 32: one row per warp at a time)
                int o = s_woff[warp], k = 0;
                for (int64_t r = (int64_t)warp * W + b; r < n; r += rstep, k++) {
                    const int len = s_rl[k * PC_WARPS + warp];
                    double sum = 0.0;
                    int j = lane;
                    for (; j + (PC_XS_UNROLL - 1) * 32 < len; j += PC_XS_UNROLL * 32) {
                        int cu[PC_XS_UNROLL];
                        double vu[PC_XS_UNROLL];
#pragma unroll
                        for (int t = 0; t < PC_XS_UNROLL; t++) { cu[t] = s_ac[o + j + t * 32]; vu[t] = s_av[o + j + t * 32]; }
#pragma unroll
                        for (int t = 0; t < PC_XS_UNROLL; t++) sum = fma(vu[t], s_xs[cu[t]], sum);
                    }
                    for (; j < len; j += 32) sum = fma(s_av[o + j], s_xs[s_ac[o + j]], sum);
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(FULL_MASK, sum, off);
                    if (lane == 0) z[r] = sum;
                    o += len;
                }
            } else
            // row groups dealt round-robin over the CTAs first (warp w of CTA b takes group
            // w W + b): consecutive rows -- similar lengths -- land on different SMs
#if PC_ROW_INTERLEAVE
            for (int64_t r0 = ((int64_t)warp * W + b) * groups; r0 < n; r0 += stride) {
#else
            for (int64_t r0 = ((int64_t)b * PC_WARPS + warp) * groups; r0 < n; r0 += stride) {
#endif
                const int64_t r = r0 + sub;
                double sum = 0.0;
                if (r < n && xs) {
                    const int64_t q1 = (int64_t)__ldg(rowptr + r + 1);
                    int64_t q = (int64_t)__ldg(rowptr + r) + sl;
#if PC_XS_PRED
                    // PC_XS_UNROLL independent loads per lane per round trip, the last round predicated
                    for (; q < q1; q += PC_XS_UNROLL * lpr) {
                        int cu[PC_XS_UNROLL];
                        double vu[PC_XS_UNROLL];
#pragma unroll
                        for (int k = 0; k < PC_XS_UNROLL; k++) {
                            const bool in = q + k * lpr < q1;
                            cu[k] = in ? (int)__ldg(col + q + k * lpr) : 0;
                            vu[k] = in ? __ldg(val + q + k * lpr) : 0.0;
                        }
#pragma unroll
                        for (int k = 0; k < PC_XS_UNROLL; k++)
                            if (q + k * lpr < q1) sum = fma(vu[k], s_xs[cu[k]], sum);
                    }
#else
                    for (; q + (PC_XS_UNROLL - 1) * lpr < q1; q += PC_XS_UNROLL * lpr) {
                        int cu[PC_XS_UNROLL];
                        double vu[PC_XS_UNROLL];
#pragma unroll
                        for (int k = 0; k < PC_XS_UNROLL; k++) { cu[k] = (int)__ldg(col + q + k * lpr); vu[k] = __ldg(val + q + k * lpr); }
#pragma unroll
                        for (int k = 0; k < PC_XS_UNROLL; k++) sum = fma(vu[k], s_xs[cu[k]], sum);
                    }
                    for (; q < q1; q += lpr) sum = fma(__ldg(val + q), s_xs[(int)__ldg(col + q)], sum);
#endif
                } else if (r < n) {
                    const int64_t q1 = (int64_t)__ldg(rowptr + r + 1);
                    int64_t q = (int64_t)__ldg(rowptr + r) + sl;
                    for (; q + 3 * lpr < q1; q += 4 * lpr) {
                        int64_t c4[4];
                        double v4[4], x4[4];
#pragma unroll
                        for (int k = 0; k < 4; k++) { c4[k] = (int64_t)__ldg(col + q + k * lpr); v4[k] = __ldg(val + q + k * lpr); }
#pragma unroll
                        for (int k = 0; k < 4; k++) x4[k] = __ldcg(u + c4[k]);
#pragma unroll
                        for (int k = 0; k < 4; k++) sum = fma(v4[k], x4[k], sum);
                    }
                    for (; q < q1; q += lpr) sum = fma(__ldg(val + q), __ldcg(u + (int64_t)__ldg(col + q)), sum);
                }
                for (int off = lpr >> 1; off > 0; off >>= 1) sum += __shfl_xor_sync(FULL_MASK, sum, off);
                if (r < n && sl == 0) z[r] = sum;
            }
            grid_barrier(flags, W, epoch);
        }
        if (b == 0) stamp(p, 1);
        // ---- B: dots [V_p, u]^T [u, z] -> d.dots + p*dld (Step 4, one reduction) ------
        if (part) {
            // larger n: CTA b owns a contiguous row block and all 2(p+1) partial dots of it
            // (u and z read once overall); after a barrier, warp i of the grid sums output i
            // over the partials in CTA order (the block dot's stage 2, spread over the grid)
            double* out = d.dots + (int64_t)p * d.dld;
            const int items = p + 1, stride = 2 * items;
            const int64_t rpb = ((n + W - 1) / W + 31) / 32 * 32;
            const int64_t rb0 = min((int64_t)b * rpb, n), rb1 = min(rb0 + rpb, n);
            // warp w: 4 columns at a time over the CTA's rows (lane = row), one butterfly for
            // the 8 sums, no block-wide synchronisation
            for (int cb = 4 * warp; cb < items; cb += 4 * PC_WARPS) {
                const int nc = min(4, items - cb);
                double a[8];
#pragma unroll
                for (int c = 0; c < 8; c++) a[c] = 0.0;
#pragma unroll 4
                for (int64_t r = rb0 + lane; r < rb1; r += 32) {
                    const double uu = __ldcg(u + r);
                    const double zz = drain ? 0.0 : __ldcg(z + r);
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        if (c < nc) {
                            const double v = __ldcg(V + (int64_t)(cb + c) * ld + r);
                            a[c] = fma(v, uu, a[c]);
                            a[4 + c] = fma(v, zz, a[4 + c]);
                        }
                    }
                }
                const double t = bfly8(a, lane);  // lane holds value lane >> 2
                const int idx = lane >> 2, c = idx & 3, which = idx >> 2;
                if ((lane & 3) == 0 && c < nc) part[(int64_t)b * stride + which * items + cb + c] = t;
            }
            grid_barrier(flags, W, epoch);
            for (int i = b * PC_WARPS + warp; i < (drain ? items : stride); i += W * PC_WARPS) {
                double t = 0.0;
                for (int q = lane; q < W; q += 32) t += __ldcg(part + (int64_t)q * stride + i);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(FULL_MASK, t, off);
                if (lane == 0) out[i] = t;  // [V_p^T u, u.u | V_p^T z, u.z]: same layout
            }
        } else {
            double* out = d.dots + (int64_t)p * d.dld;
            const int items = p + 1;
            const int per = (items + W - 1) / W;
            const int c0 = b * per, c1 = min(c0 + per, items);
            for (int cb = c0; cb < c1; cb += PC_CB) {
                const int nc = min(PC_CB, c1 - cb);
                double au[PC_CB], az[PC_CB];
#pragma unroll
                for (int c = 0; c < PC_CB; c++) { au[c] = 0.0; az[c] = 0.0; }
                for (int64_t r = tid; r < n; r += PC_THREADS) {
                    const double uu = __ldcg(u + r);
                    const double zz = drain ? 0.0 : __ldcg(z + r);
#pragma unroll
                    for (int c = 0; c < PC_CB; c++) {
                        if (c < nc) {
                            const double v = __ldcg(V + (int64_t)(cb + c) * ld + r);
                            au[c] = fma(v, uu, au[c]);
                            az[c] = fma(v, zz, az[c]);
                        }
                    }
                }
                static_assert(PC_CB == 8, "bfly8 reduces 8 columns");
                const double ru = bfly8(au, lane);  // lane holds column lane >> 2
                const double rz = bfly8(az, lane);
                if ((lane & 3) == 0) {
                    s_red[warp * 2 * PC_CB + (lane >> 2)] = ru;
                    s_red[warp * 2 * PC_CB + PC_CB + (lane >> 2)] = rz;
                }
                __syncthreads();
                if (tid < 2 * nc) {
                    const int c = tid % nc, which = tid / nc;  // 0: V_c.u, 1: V_c.z
                    double t = 0.0;
                    for (int w = 0; w < PC_WARPS; w++) t += s_red[w * 2 * PC_CB + which * PC_CB + c];
                    if (which == 0) out[cb + c] = t;
                    else if (!drain) out[p + 1 + cb + c] = t;
                }
                __syncthreads();
            }
        }
        grid_barrier(flags, W, epoch);
        if (b == 0) stamp(p, 2);
        if (gs == 2 && split && b == 0 && tid == 0) { __threadfence(); st_release_u32(flags + 5, (unsigned)p); }  // dots of p final
        // ---- C: critical small step ----------------------------------------------------------
        // Alg. 3 (gs = 2): every worker computes the critical step from the same reduced dots
        // (bitwise the coefficients CTA 0 publishes for the tail), so no barrier separates it
        // from the update; the stop decision is uniform: a stop the tail recorded at an
        // iteration <= p - PC_LAG (final once tail_done >= p - PC_LAG).  Alg. 2 one sweep:
        // CTA 0 (its forward substitution reads L rows other CTAs do not have), a barrier.
        bool local_coef = false;
        if (gs == 2) {
            if (tid == 0) {
                if (split && p > PC_LAG)
                    while (ld_acquire_u32(flags + 3) < (unsigned)(p - PC_LAG)) {
                    }
                if (b == 0 && prof) {  // IGS_PC_PROF: end of the wait for TAIL(p - PC_LAG)
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    prof[(int64_t)(m + 2) * 8 + (int64_t)p * 8 + 6] = t;
                }
                int go;
                if (split) {
                    const unsigned sa = ld_acquire_u32(flags + 4);
                    go = !(sa != 0u && (int)sa <= p - PC_LAG);
                } else {
                    go = (vist[ST_STATUS] == RUNNING);
                }
                s_go = go;
                if (!go && b == 0) { __threadfence(); st_release_u32(flags + 2, (unsigned)p); }
                s_coef[1] = 0.0;  // mode 0 unless the critical step below completes
            }
            __syncthreads();
            if (!s_go) break;
            small_body(d, SS_CRIT, gs, p, m, s_small, red, /*publish=*/!split, /*loc=*/s_coef);
            __syncthreads();
            if (b == 0) { stamp(p, 3); stamp(p, 4); }
            local_coef = true;
        } else {
            if (b == 0) {
                if (tid == 0) {
                    if (split && p > PC_LAG)
                        while (ld_acquire_u32(flags + 3) < (unsigned)(p - PC_LAG)) {
                        }
                    s_go = (vist[ST_STATUS] == RUNNING);
                    if (!s_go) { __threadfence(); st_release_u32(flags + 2, (unsigned)p); }
                }
                __syncthreads();
                if (s_go) {
                    small_body(d, SS_CRIT, gs, p, m, s_small, red, true, nullptr, false,
                               prof ? prof + (int64_t)(m + 2) * 16 + (int64_t)p * 8 : nullptr);
                    __syncthreads();
                    if (tid == 0) { __threadfence(); st_release_u32(flags + 1, (unsigned)p); }
                }
                stamp(p, 3);
            }
            grid_barrier(flags, W, epoch);
            if (b == 0) stamp(p, 4);
            if (*(volatile unsigned*)(flags + 2) != 0u) break;  // uniform: written before the barrier
        }
        // ---- D: fused update (Steps 10-13) -------------------------------------------------
        {
            int mode = local_coef ? (int)s_coef[1] : ((vist[ST_MODE_IT] == p) ? vist[ST_MODE] : 0);
            mode &= drain ? 1 : 3;
            if (mode != 0) {
                const bool want_next = (mode & 2) != 0;
                // local: alpha = r2 in small_body's s_a, [gamma, mode, beta...] in s_coef
                double* sa = local_coef ? s_small : s_coef;
                double* sbt = local_coef ? s_coef + 2 : s_coef + (M + 1);
                if (!local_coef) {
                    if (gs == 2)
                        for (int j = tid; j < p; j += PC_THREADS) sa[j] = __ldcg(d.alpha + j);
                    if (want_next)
                        for (int j = tid; j <= p; j += PC_THREADS) sbt[j] = __ldcg(d.beta + j);
                }
                const double gamma = local_coef ? s_coef[0] : __ldcg(d.scal + SC_GAMMA);
                __syncthreads();
                double* r1s = s_red;                  // [PC_WARPS][32]
                double* r2s = s_red + PC_WARPS * 32;  // [PC_WARPS][32]
                const int64_t ntiles = (n + 31) / 32;
                const int64_t mine = ntiles > b ? (ntiles - b + W - 1) / W : 0;  // tiles b, b+W, ...
                for (int64_t g0 = 0; g0 < mine; g0 += PC_WARPS) {
                    const int nt = (int)min((int64_t)PC_WARPS, mine - g0);
                    const int S = PC_WARPS / nt;  // warps (column slices) per tile
                    const int ti = warp / S, sl = warp % S;
                    double t1 = 0.0, t2 = 0.0, uu = 0.0, zz = 0.0;
                    if (warp < nt) {  // the epilogue's u and z, fetched ahead of the column loop
                        const int64_t r = (b + (g0 + warp) * W) * 32 + lane;
                        if (r < n) { uu = __ldcg(u + r); if (want_next) zz = __ldcg(z + r); }
                    }
                    if (ti < nt) {
                        const int64_t r = (b + (g0 + ti) * W) * 32 + lane;
                        if (r < n) {
#pragma unroll 8
                            for (int j = sl; j < p; j += S) {
                                const double v = __ldcg(V + (int64_t)j * ld + r);
                                if (gs == 2) t1 = fma(v, sa[j], t1);
                                if (want_next) t2 = fma(v, sbt[j], t2);
                            }
                        }
                    }
                    r1s[warp * 32 + lane] = t1;
                    r2s[warp * 32 + lane] = t2;
                    __syncthreads();
                    if (warp < nt) {
                        const int64_t r = (b + (g0 + warp) * W) * 32 + lane;
                        if (r < n) {
                            double s1 = 0.0, s2 = 0.0;
                            for (int k = 0; k < S; k++) { s1 += r1s[(warp * S + k) * 32 + lane]; s2 += r2s[(warp * S + k) * 32 + lane]; }
                            const double w_ = (gs == 2) ? uu - s1 : uu;
                            const double vv = w_ / gamma;
                            if (want_next) V[(int64_t)(p + 1) * ld + r] = zz / gamma - fma(vv, sbt[p], s2);
                            if (mode & 1) V[(int64_t)p * ld + r] = vv;
                        }
                    }
                    __syncthreads();
                }
            }
        }
        if (b == 0) stamp(p, 5);
        if (!split) {  // one CTA: the tail runs in line
            if (tid == 0 && vist[ST_STATUS] == RUNNING) counter[1] += 1u;
            __syncthreads();
            stamp(p, 6);
            small_body(d, SS_TAIL, gs, p, m, s_small, red, true, nullptr, /*r3_ready=*/tri,
                       prof ? prof + (int64_t)(m + 2) * 8 + (int64_t)p * 8 : nullptr);
            stamp(p, 7);
        }
        grid_barrier(flags, W, epoch);
    }
}

static size_t pcycle_smem(int M) {
    return small_smem(M) + (size_t)(2 * (M + 1) + 2 * PC_WARPS * 32) * sizeof(double);
}

int64_t pcycle_xs_max() { return 8192; }  // staged u: <= 64 KB of shared memory

template <typename IT, typename PT>
static cudaError_t pcycle_go(const Dev& d, const SpmvArgs& a, double* V, int64_t ld, double* z, int64_t n,
                             int m, int gs, unsigned* flags, unsigned* counter, int grid, cudaStream_t s,
                             unsigned long long* prof, double* part, int xs, int ntri, int* ares_io) {
    auto fn = pcycle_kernel<IT, PT>;
    int ares = ares_io ? *ares_io : 0;
    // resident A (xs only): values + 16-bit columns of the CTA's rows + its warps' row lengths
    const int W = pcycle_worker_ctas(grid, gs, ntri);
    const size_t base = pcycle_smem(d.m) + (xs ? (size_t)n * sizeof(double) : 0);
    auto ares_bytes = [&](int a) {
        const int64_t K = (n + (int64_t)W * PC_WARPS - 1) / ((int64_t)W * PC_WARPS);
        return (size_t)a * 8 + (size_t)((a + 3) & ~3) * 2 + (size_t)(PC_WARPS * K) * sizeof(int);
    };
    if (!xs || a.lpr != 32 || n > 65535 || ares <= 0 || base + ares_bytes(ares) > 227 * 1024) ares = 0;
    const size_t smem = base + (ares ? ares_bytes(ares) : 0);
    if (ares_io) *ares_io = ares;  // what the launch uses
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, PC_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
    Dev dd = d;
    const PT* rp = static_cast<const PT*>(a.rowptr);
    const IT* ci = static_cast<const IT*>(a.col);
    const double* va = a.val;
    int lpr = a.lpr > 0 ? a.lpr : 4;
    SellDev<IT> sell = sell_dev<IT>(a);
    void* args[] = {&dd, &n, &m, &gs, (void*)&rp, (void*)&ci, (void*)&va, &lpr, &V, &ld, &z, &flags, &counter, &prof,
                    &part, (void*)&sell, &xs, &ntri, &ares};
    return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(PC_THREADS), args, smem, s);
}

int pcycle_max_grid(int num_sms) { return num_sms; }

int pcycle_worker_ctas(int grid, int gs, int ntri) {
    const int nt = (gs == 2 && grid >= 3) ? std::max(1, std::min(ntri, grid - 2)) : 0;
    return grid > 1 ? grid - 1 - nt : 1;
}
static_assert(PCYCLE_WARPS == PC_WARPS, "igs_internal.cuh: PCYCLE_WARPS");

cudaError_t launch_pcycle(const Dev& d, const SpmvArgs& a, double* V, int64_t ld, double* z, int64_t n,
                          int m, int gs, unsigned* flags, unsigned* counter, int grid, cudaStream_t s,
                          unsigned long long* prof, double* part, int xs, int ntri, int* ares) {
    if (a.idx64) {
        if (a.ptr64) return pcycle_go<int64_t, int64_t>(d, a, V, ld, z, n, m, gs, flags, counter, grid, s, prof, part, xs, ntri, ares);
        return pcycle_go<int64_t, int32_t>(d, a, V, ld, z, n, m, gs, flags, counter, grid, s, prof, part, xs, ntri, ares);
    }
    if (a.ptr64) return pcycle_go<int32_t, int64_t>(d, a, V, ld, z, n, m, gs, flags, counter, grid, s, prof, part, xs, ntri, ares);
    return pcycle_go<int32_t, int32_t>(d, a, V, ld, z, n, m, gs, flags, counter, grid, s, prof, part, xs, ntri, ares);
}

}  // namespace igs
