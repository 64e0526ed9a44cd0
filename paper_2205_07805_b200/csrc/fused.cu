// fused.cu -- one persistent wavefront kernel per Arnoldi iteration (single GPU):
//
//     fused update of iteration p      v_p = (u - V_p r2)/gamma, u' = z/gamma - V_{p+1} r1
//   + SpMV of iteration p+1            z' = A u'
//   + fused block dot of iteration p+1 [V_{p+1}, u']^T [u', z']
//
// The unfused path streams V_p from HBM twice per iteration (update, then block dot one
// SpMV later).  Here the SpMV's dependence on u' is only a band of `reach` rows (one grid
// plane for the 3D stencil), so tile s can run its SpMV + block dot as soon as the update
// of tiles s-L..s+L (L = ceil(reach/T)) is done: phase B(s) trails phase A by L+1 tiles,
// and the V rows phase A just streamed are re-read from the 126 MB L2 instead of HBM.  HBM
// traffic per iteration drops from 2 x 8np + A to 8np + A (SURVEY §8(d) byte model counts
// two reads of V_p).  Phase A publishes per-tile flags (release); phase B waits for its
// neighbourhood (acquire).  Work item w (static round robin over the co-resident grid):
// A(w), then B(w - L - 1).  Phase B loads of data written in this kernel use ld.global.cg.
//
// Determinism: each lane accumulates its rows' dot contributions in a fixed order (tiles in
// CTA order), one warp reduction per column at the end, per-CTA partials summed in CTA
// order by the last CTA -- bitwise reproducible run to run.
//
// P:n = PAPER.md line n.  Alg. 3 Steps 10-13 and Step 4.
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_internal.cuh"

namespace igs {

#define FULL_MASK 0xffffffffu
constexpr int FU_T = 128;        // rows per tile
constexpr int FU_THREADS = 256;  // 8 warps
constexpr int FU_WARPS = 8;
constexpr int FU_K = 8;          // staged SpMV nonzeros per thread (cap 2048 per tile)

__device__ __forceinline__ double2 ldcg2(const double* p) {
    return __ldcg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 ld2_any(const double* __restrict__ p, int64_t r, int64_t n, bool cg) {
    if (r + 1 < n) return cg ? ldcg2(p + r) : __ldg(reinterpret_cast<const double2*>(p + r));
    double2 v;
    v.x = (r < n) ? (cg ? __ldcg(p + r) : __ldg(p + r)) : 0.0;
    v.y = 0.0;
    return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ long long ld_acquire64(const long long* p) {
    long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release64(long long* p, long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct FusedArgs {
    int64_t n;
    int p;                 // iteration whose update runs (normalised columns 0..p-1)
    int m;                 // cycle length (p + 1 == m -> drain: no SpMV in phase B)
    const double* V;
    int64_t ld;
    double* z;             // in: A u (iteration p); out: A u' (iteration p+1)
    const double* alpha;   // r2 (Alg. 3) or NULL (Alg. 2)
    const double* beta;    // r1, p+1 entries
    const double* gamma;   // device scalar
    const void* rowptr;
    const void* col;
    const double* val;
    int lag;               // L + 1 tiles
    long long* progress;   // per CTA: (epoch << 32) | (last tile whose phase A finished) + 1
    int epoch;
    double* part;          // [grid * 2 (p+2)]
    double* out;           // dots of iteration p+1
    unsigned* counter;
    const int* istate;
};

template <int MAXG, bool NV2, bool HAS_ALPHA, typename IT, typename PT>
__global__ void __launch_bounds__(FU_THREADS, 2) fused_kernel(FusedArgs a) {
    const int* ist = a.istate;
    {
        const volatile int* vs = ist;
        if (vs[ST_MODE_IT] != a.p || vs[ST_MODE] != 3) return;  // stopped / breakdown
    }
    extern __shared__ double fsm[];
    const int p = a.p;
    const int ncols = p + 2;                      // V_0..V_p and u' itself
    double* s_alpha = fsm;                        // [p]
    double* s_beta = s_alpha + (p + 1);           // [p+1]
    double* s_red = s_beta + (p + 2);             // [8][128][2]
    double* s_prod = s_red + FU_WARPS * FU_T * 2; // [FU_K * 256]
    double* s_z = s_prod + FU_K * FU_THREADS;     // [128]
    double* s_acc = s_z + FU_T;                   // [2 * ncols]
    __shared__ bool s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < p; j += FU_THREADS) s_alpha[j] = HAS_ALPHA ? a.alpha[j] : 0.0;
    for (int j = tid; j <= p; j += FU_THREADS) s_beta[j] = a.beta[j];
    const double gamma = *a.gamma;
    __syncthreads();

    const int64_t n = a.n;
    const int64_t ld = a.ld;
    const double* __restrict__ V = a.V;
    double* u = const_cast<double*>(V) + (int64_t)p * ld;        // pending -> v_p in place
    double* un = const_cast<double*>(V) + (int64_t)(p + 1) * ld; // u'
    const PT* __restrict__ rowptr = static_cast<const PT*>(a.rowptr);
    const IT* __restrict__ col = static_cast<const IT*>(a.col);
    const bool drain = (p + 1 == a.m);
    const int64_t ntiles = (n + FU_T - 1) / FU_T;
    const int64_t nitems = ntiles + a.lag;

    double accu[MAXG], accz[MAXG];
#pragma unroll
    for (int g = 0; g < MAXG; g++) { accu[g] = 0.0; accz[g] = 0.0; }

    for (int64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
        // ================= phase A: update of tile w =================
        if (w < ntiles) {
            const int64_t r0 = w * FU_T;
            const int64_t ra = r0 + 2 * lane, rb = ra + 64;
            double2 t1a = make_double2(0.0, 0.0), t1b = t1a, t2a = t1a, t2b = t1a;
            for (int j0 = warp; j0 < p; j0 += 8 * FU_WARPS) {
                double2 va[8], vb[8];
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const int j = j0 + c * FU_WARPS;
                    if (j < p) {
                        va[c] = ld2_any(V + (int64_t)j * ld, ra, n, false);
                        vb[c] = ld2_any(V + (int64_t)j * ld, rb, n, false);
                    } else {
                        va[c] = make_double2(0.0, 0.0);
                        vb[c] = va[c];
                    }
                }
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const int j = j0 + c * FU_WARPS;
                    const double al = j < p ? s_alpha[j] : 0.0, be = j < p ? s_beta[j] : 0.0;
                    if (HAS_ALPHA) {
                        t1a.x = fma(va[c].x, al, t1a.x); t1a.y = fma(va[c].y, al, t1a.y);
                        t1b.x = fma(vb[c].x, al, t1b.x); t1b.y = fma(vb[c].y, al, t1b.y);
                    }
                    t2a.x = fma(va[c].x, be, t2a.x); t2a.y = fma(va[c].y, be, t2a.y);
                    t2b.x = fma(vb[c].x, be, t2b.x); t2b.y = fma(vb[c].y, be, t2b.y);
                }
            }
            double* rw = s_red + warp * FU_T * 2;
            rw[2 * (2 * lane)] = t1a.x;      rw[2 * (2 * lane) + 1] = t2a.x;
            rw[2 * (2 * lane + 1)] = t1a.y;  rw[2 * (2 * lane + 1) + 1] = t2a.y;
            rw[2 * (64 + 2 * lane)] = t1b.x; rw[2 * (64 + 2 * lane) + 1] = t2b.x;
            rw[2 * (65 + 2 * lane)] = t1b.y; rw[2 * (65 + 2 * lane) + 1] = t2b.y;
            __syncthreads();
            if (tid < FU_T) {
                const int64_t r = r0 + tid;
                if (r < n) {
                    double T1 = 0.0, T2 = 0.0;
#pragma unroll
                    for (int ww = 0; ww < FU_WARPS; ww++) {
                        T1 += s_red[(ww * FU_T + tid) * 2];
                        T2 += s_red[(ww * FU_T + tid) * 2 + 1];
                    }
                    const double uu = u[r];
                    const double v = (HAS_ALPHA ? uu - T1 : uu) / gamma;
                    const double zz = a.z[r];
                    u[r] = v;
                    un[r] = zz / gamma - fma(v, s_beta[p], T2);
                }
            }
            __threadfence();
            __syncthreads();
            // progress word of this CTA: its tiles finish in increasing order, so
            // "progress >= (epoch, t+1)" means every tile <= t it owns is done
            if (tid == 0) st_release64(a.progress + blockIdx.x, ((long long)a.epoch << 32) | (long long)(w + 1));
        }
        // ================= phase B: SpMV + block dot of tile s =================
        const int64_t s = w - a.lag;
        if (s >= 0 && s < ntiles) {
            const int64_t r0 = s * FU_T;
            // wait for the update of every tile the SpMV of tile s can touch
            const int64_t t0 = s - a.lag + 1 > 0 ? s - a.lag + 1 : 0;
            const int64_t t1 = s + a.lag - 1 < ntiles - 1 ? s + a.lag - 1 : ntiles - 1;
            {
                const int64_t G = gridDim.x;
                const int64_t span = t1 - t0 + 1;
                for (int64_t k = tid; k < (span < G ? span : G); k += FU_THREADS) {
                    // owner of tile t is t % G; the newest tile <= t1 it owns
                    const int64_t owner = (t1 - k) % G;
                    const int64_t need = ((long long)a.epoch << 32) | (long long)(t1 - k + 1);
                    while (ld_acquire64(a.progress + owner) < need) __nanosleep(32);
                }
            }
            __syncthreads();
            const int64_t rl = r0 + FU_T < n ? r0 + FU_T : n;
            if (!drain) {
                const int64_t q0 = (int64_t)__ldg(rowptr + r0), q1 = (int64_t)__ldg(rowptr + rl);
                const int cnt = (int)(q1 - q0);
                if (cnt <= FU_K * FU_THREADS) {
                    int64_t cc[FU_K];
                    double vv[FU_K], xv[FU_K];
#pragma unroll
                    for (int k = 0; k < FU_K; k++) {
                        const int i = tid + k * FU_THREADS;
                        cc[k] = i < cnt ? (int64_t)__ldg(col + q0 + i) : 0;
                        vv[k] = i < cnt ? __ldg(a.val + q0 + i) : 0.0;
                    }
#pragma unroll
                    for (int k = 0; k < FU_K; k++) xv[k] = (tid + k * FU_THREADS < cnt) ? __ldcg(un + cc[k]) : 0.0;
#pragma unroll
                    for (int k = 0; k < FU_K; k++) {
                        const int i = tid + k * FU_THREADS;
                        if (i < cnt) s_prod[i] = __dmul_rn(vv[k], xv[k]);
                    }
                    __syncthreads();
                    if (tid < FU_T) {
                        const int64_t r = r0 + tid;
                        double sum = 0.0;
                        if (r < n) {
                            const int q_a = (int)((int64_t)__ldg(rowptr + r) - q0);
                            const int q_e = (int)((int64_t)__ldg(rowptr + r + 1) - q0);
                            for (int q = q_a; q < q_e; q++) sum = __dadd_rn(sum, s_prod[q]);
                            a.z[r] = sum;
                        }
                        s_z[tid] = sum;
                    }
                } else if (tid < FU_T) {
                    const int64_t r = r0 + tid;
                    double sum = 0.0;
                    if (r < n) {
                        for (int64_t q = __ldg(rowptr + r); q < (int64_t)__ldg(rowptr + r + 1); q++)
                            sum = __dadd_rn(sum, __dmul_rn(__ldg(a.val + q), __ldcg(un + __ldg(col + q))));
                        a.z[r] = sum;
                    }
                    s_z[tid] = sum;
                }
                __syncthreads();
            }
            // block dot rows: lane owns rows {2l, 2l+1, 64+2l, 65+2l} of the tile
            const int64_t ra = r0 + 2 * lane, rb = ra + 64;
            const double2 ua = ld2_any(un, ra, n, true), ub = ld2_any(un, rb, n, true);
            double2 za = make_double2(0.0, 0.0), zb = za;
            if (NV2 && !drain) {
                za = make_double2(s_z[2 * lane], s_z[2 * lane + 1]);
                zb = make_double2(s_z[64 + 2 * lane], s_z[65 + 2 * lane]);
                if (ra >= n) za.x = 0.0;
                if (ra + 1 >= n) za.y = 0.0;
                if (rb >= n) zb.x = 0.0;
                if (rb + 1 >= n) zb.y = 0.0;
            }
#pragma unroll
            for (int g = 0; g < MAXG; g++) {
                const int j = g * FU_WARPS + warp;
                if (j < ncols) {
                    double2 va, vb;
                    if (j <= p) {
                        va = ld2_any(V + (int64_t)j * ld, ra, n, true);
                        vb = ld2_any(V + (int64_t)j * ld, rb, n, true);
                    } else {
                        va = ua;
                        vb = ub;
                    }
                    accu[g] = fma(vb.y, ub.y, fma(vb.x, ub.x, fma(va.y, ua.y, fma(va.x, ua.x, accu[g]))));
                    if (NV2) accz[g] = fma(vb.y, zb.y, fma(vb.x, zb.x, fma(va.y, za.y, fma(va.x, za.x, accz[g]))));
                }
            }
            __syncthreads();  // s_z / s_prod reused by the next item
        }
    }
    // ================= per-CTA partials, last CTA reduces in CTA order =================
    const int stride = (NV2 && !drain) ? 2 * ncols : ncols;
#pragma unroll
    for (int g = 0; g < MAXG; g++) {
        const int j = g * FU_WARPS + warp;
        double su = accu[g], sz = accz[g];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            su += __shfl_xor_sync(FULL_MASK, su, off);
            sz += __shfl_xor_sync(FULL_MASK, sz, off);
        }
        if (lane == 0 && j < ncols) {
            s_acc[j] = su;
            if (NV2 && !drain) s_acc[ncols + j] = sz;
        }
    }
    __syncthreads();
    for (int i = tid; i < stride; i += FU_THREADS) a.part[(int64_t)blockIdx.x * stride + i] = s_acc[i];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int i = tid; i < stride; i += FU_THREADS) {
        double sacc = 0.0;
        for (int bb = 0; bb < (int)gridDim.x; bb++) sacc += __ldcg(a.part + (int64_t)bb * stride + i);
        a.out[i] = sacc;
    }
    if (tid == 0) *a.counter = 0u;
}

static size_t fused_smem(int p) {
    return (size_t)((p + 1) + (p + 2) + FU_WARPS * FU_T * 2 + FU_K * FU_THREADS + FU_T + 2 * (p + 2) + 8) * sizeof(double);
}

template <int MAXG, bool NV2, bool HA, typename IT, typename PT>
static cudaError_t fused_go(const FusedArgs& a, int grid, cudaStream_t s) {
    auto k = fused_kernel<MAXG, NV2, HA, IT, PT>;
    const size_t smem = fused_smem(a.p);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, FU_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

template <int MAXG, typename IT, typename PT>
static cudaError_t fused_g(const FusedArgs& a, int grid, bool has_alpha, cudaStream_t s) {
    const bool nv2 = (a.p + 1 != a.m);
    if (has_alpha) return nv2 ? fused_go<MAXG, true, true, IT, PT>(a, grid, s) : fused_go<MAXG, false, true, IT, PT>(a, grid, s);
    return nv2 ? fused_go<MAXG, true, false, IT, PT>(a, grid, s) : fused_go<MAXG, false, false, IT, PT>(a, grid, s);
}

template <typename IT, typename PT>
static cudaError_t fused_t(const FusedArgs& a, int grid, bool has_alpha, cudaStream_t s) {
    const int ncols = a.p + 2;
    if (ncols <= 4 * FU_WARPS) return fused_g<4, IT, PT>(a, grid, has_alpha, s);
    if (ncols <= 8 * FU_WARPS) return fused_g<8, IT, PT>(a, grid, has_alpha, s);
    return fused_g<16, IT, PT>(a, grid, has_alpha, s);
}

int fused_max_cols() { return 16 * FU_WARPS; }
int fused_tile_rows() { return FU_T; }

int fused_grid(int num_sms) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_kernel<16, true, true, int32_t, int32_t>,
                                                  FU_THREADS, fused_smem(120));
    if (occ < 1) occ = 1;
    return num_sms * occ;
}

cudaError_t launch_fused(int64_t n, int p, int m, const double* V, int64_t ld, double* z,
                         const double* alpha, const double* beta, const double* gamma_dev,
                         const SpmvArgs& A, int lag, long long* progress, int epoch, double* part,
                         double* out, unsigned* counter, const int* istate, int grid,
                         cudaStream_t s) {
    FusedArgs a{n, p, m, V, ld, z, alpha, beta, gamma_dev, A.rowptr, A.col, A.val, lag, progress, epoch,
                part, out, counter, istate};
    if (A.idx64) return A.ptr64 ? fused_t<int64_t, int64_t>(a, grid, alpha != nullptr, s)
                                : fused_t<int64_t, int32_t>(a, grid, alpha != nullptr, s);
    return A.ptr64 ? fused_t<int32_t, int64_t>(a, grid, alpha != nullptr, s)
                   : fused_t<int32_t, int32_t>(a, grid, alpha != nullptr, s);
}

}  // namespace igs
