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
#include "ptx_util.cuh"

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

__device__ __forceinline__ void named_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(FU_THREADS) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ld2_pol(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld2_cg_pol(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol) : "memory");
    return v;
}
// guarded 2-row load with an L2 policy (rows r, r+1 of a column; zero beyond n)
__device__ __forceinline__ double2 ld2_rows(const double* col, int64_t r, int64_t n, bool cg, uint64_t pol) {
    if (r + 1 < n) return cg ? ld2_cg_pol(col + r, pol) : ld2_pol(col + r, pol);
    double2 v;
    v.x = (r < n) ? __ldcg(col + r) : 0.0;
    v.y = 0.0;
    return v;
}

// CTA = 17 warps:
//   warps 0-7   phase A consumers: update of the CTA's tiles c, c+G, ... from a shared-memory
//               ring (warp w owns column 8g+w of column group g; cross-warp sum per row);
//   warp 8      producer: streams V_p (8 columns x 128 rows per stage, cp.async.bulk with an
//               L2 evict_last hint) into a 16-stage ring -- HBM never waits for the math;
//   warps 9-16  phase B: SpMV + block dot of the same tiles once their neighbourhood is
//               updated (V re-read from L2, evict_first).
// The producer may run at most `ahead` own tiles in front of phase B (bounds the L2 window);
// phase B waits on the per-CTA global progress words of the neighbourhood's owners.
constexpr int FU_STAGES = 16;
constexpr int FU_STAGE_D = FU_WARPS * FU_T;   // 8 columns x 128 rows = 8 KB
constexpr int FU_CTA_THREADS = 2 * FU_THREADS + 32;

template <int MAXG, bool NV2, bool HAS_ALPHA, typename IT, typename PT>
__global__ void __launch_bounds__(FU_CTA_THREADS, 1) fused_kernel(FusedArgs a) {
    const int* ist = a.istate;
    {
        const volatile int* vs = ist;
        if (vs[ST_MODE_IT] != a.p || vs[ST_MODE] != 3) return;  // stopped / breakdown
    }
    extern __shared__ __align__(128) double fsm[];
    const int p = a.p;
    const int ncols = p + 2;                      // V_0..V_p and u' itself
    double* ring = fsm;                           // [STAGES][8][128]
    double* s_red = ring + FU_STAGES * FU_STAGE_D;   // [8][128][2]   (A consumers)
    double* s_prod = s_red + FU_WARPS * FU_T * 2;    // [FU_K * 256]  (B)
    double* s_z = s_prod + FU_K * FU_THREADS;        // [128]         (B)
    double* s_alpha = s_z + FU_T;                    // [p]
    double* s_beta = s_alpha + (p + 1);              // [p+1]
    double* s_acc = s_beta + (p + 2);                // [2 * ncols]
    uint64_t* full = reinterpret_cast<uint64_t*>(s_acc + 2 * ncols + 2);
    uint64_t* empty = full + FU_STAGES;
    __shared__ bool s_last;
    __shared__ volatile int s_bdone;              // own tiles finished by phase B
    const int tid = threadIdx.x;
    const int role = tid < FU_THREADS ? 0 : (tid < FU_THREADS + 32 ? 1 : 2);  // A, producer, B
    const int gtid = role == 0 ? tid : (role == 1 ? tid - FU_THREADS : tid - FU_THREADS - 32);
    const int lane = gtid & 31, warp = gtid >> 5;
    for (int j = tid; j < p; j += FU_CTA_THREADS) s_alpha[j] = HAS_ALPHA ? a.alpha[j] : 0.0;
    for (int j = tid; j <= p; j += FU_CTA_THREADS) s_beta[j] = a.beta[j];
    if (tid == 0) {
        s_bdone = 0;
        for (int i = 0; i < FU_STAGES; i++) { mbar_init(full + i, 1); mbar_init(empty + i, FU_WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
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
    const int64_t G = gridDim.x;
    const int64_t nown = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
    const int L = a.lag;
    const int ahead = (int)((L + G - 1) / G) + 2;
    const int ngroups = (p + FU_WARPS - 1) / FU_WARPS;

    double accu[MAXG], accz[MAXG];
#pragma unroll
    for (int g = 0; g < MAXG; g++) { accu[g] = 0.0; accz[g] = 0.0; }

    if (role == 1) {
        // ============================ producer ============================
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();
            uint32_t it = 0;
            for (int64_t k = 0; k < nown; k++) {
                while (s_bdone < k - ahead) __nanosleep(200);
                const int64_t r0 = (blockIdx.x + k * G) * FU_T;
                const int64_t rows = n - r0 < FU_T ? n - r0 : FU_T;
                const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * sizeof(double));
                for (int g = 0; g < ngroups; g++, it++) {
                    const int st = it % FU_STAGES;
                    mbar_wait(empty + st, ((it / FU_STAGES) & 1) ^ 1);
                    const int c0 = g * FU_WARPS;
                    const int nc = min(FU_WARPS, p - c0);
                    mbar_arrive_expect_tx(full + st, (uint32_t)nc * bytes);
                    for (int c = 0; c < nc; c++)
                        bulk_g2s_hint(ring + (size_t)st * FU_STAGE_D + c * FU_T, V + (int64_t)(c0 + c) * ld + r0,
                                  bytes, full + st, keep);
                }
            }
        }
    } else if (role == 0) {
        // ============================ phase A consumers ============================
        uint32_t it = 0;
        for (int64_t k = 0; k < nown; k++) {
            const int64_t w = blockIdx.x + k * G;
            const int64_t r0 = w * FU_T;
            const bool fullt = r0 + FU_T <= n;
            double pu = 0.0, pz = 0.0;
            if (gtid < FU_T && r0 + gtid < n) { pu = __ldcg(u + r0 + gtid); pz = __ldcg(a.z + r0 + gtid); }
            double t1[4] = {0.0, 0.0, 0.0, 0.0}, t2[4] = {0.0, 0.0, 0.0, 0.0};
            for (int g = 0; g < ngroups; g++, it++) {
                const int st = it % FU_STAGES;
                const int c = g * FU_WARPS + warp;
                mbar_wait(full + st, (it / FU_STAGES) & 1);
                if (c < p) {
                    const double* cs = ring + (size_t)st * FU_STAGE_D + warp * FU_T;
                    const double al = s_alpha[c], be = s_beta[c];
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        double v = cs[lane + 32 * i];
                        if (!fullt && r0 + lane + 32 * i >= n) v = 0.0;
                        if (HAS_ALPHA) t1[i] = fma(v, al, t1[i]);
                        t2[i] = fma(v, be, t2[i]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + st);
            }
            double* rw = s_red + warp * FU_T * 2;
#pragma unroll
            for (int i = 0; i < 4; i++) { rw[2 * (lane + 32 * i)] = t1[i]; rw[2 * (lane + 32 * i) + 1] = t2[i]; }
            named_bar(1);
            if (gtid < FU_T) {
                const int64_t r = r0 + gtid;
                if (r < n) {
                    double T1 = 0.0, T2 = 0.0;
#pragma unroll
                    for (int ww = 0; ww < FU_WARPS; ww++) {
                        T1 += s_red[(ww * FU_T + gtid) * 2];
                        T2 += s_red[(ww * FU_T + gtid) * 2 + 1];
                    }
                    const double v = (HAS_ALPHA ? pu - T1 : pu) / gamma;
                    u[r] = v;
                    un[r] = pz / gamma - fma(v, s_beta[p], T2);
                }
            }
            named_bar(1);  // orders the stores above before thread 0's fence (cumulativity)
            if (gtid == 0) {
                __threadfence();
                st_release64(a.progress + blockIdx.x, ((long long)a.epoch << 32) | (long long)(w + 1));
            }
        }
    } else {
        // =================== phase B: SpMV + block dot (trailing) ===================
        const uint64_t drop = policy_evict_first();
        for (int64_t k = 0; k < nown; k++) {
            const int64_t s = blockIdx.x + k * G;
            const int64_t r0 = s * FU_T;
            // neighbourhood [s-L, s+L]: owner of tile t is t % G and finishes its tiles in order
            const int64_t t0 = s - L > 0 ? s - L : 0;
            const int64_t t1 = s + L < ntiles - 1 ? s + L : ntiles - 1;
            const int64_t span = t1 - t0 + 1;
            for (int64_t q = gtid; q < (span < G ? span : G); q += FU_THREADS) {
                const int64_t owner = (t1 - q) % G;
                const long long need = ((long long)a.epoch << 32) | (long long)(t1 - q + 1);
                while (ld_acquire64(a.progress + owner) < need) __nanosleep(64);
            }
            named_bar(2);
            const int64_t rl = r0 + FU_T < n ? r0 + FU_T : n;
            if (!drain) {
                const int64_t q0 = (int64_t)__ldg(rowptr + r0), q1 = (int64_t)__ldg(rowptr + rl);
                const int cnt = (int)(q1 - q0);
                if (cnt <= FU_K * FU_THREADS) {
                    int64_t cc[FU_K];
                    double vv[FU_K], xv[FU_K];
#pragma unroll
                    for (int kk = 0; kk < FU_K; kk++) {
                        const int i = gtid + kk * FU_THREADS;
                        cc[kk] = i < cnt ? (int64_t)__ldg(col + q0 + i) : 0;
                        vv[kk] = i < cnt ? __ldg(a.val + q0 + i) : 0.0;
                    }
#pragma unroll
                    for (int kk = 0; kk < FU_K; kk++) xv[kk] = (gtid + kk * FU_THREADS < cnt) ? __ldcg(un + cc[kk]) : 0.0;
#pragma unroll
                    for (int kk = 0; kk < FU_K; kk++) {
                        const int i = gtid + kk * FU_THREADS;
                        if (i < cnt) s_prod[i] = __dmul_rn(vv[kk], xv[kk]);
                    }
                    named_bar(2);
                    if (gtid < FU_T) {
                        const int64_t r = r0 + gtid;
                        double sum = 0.0;
                        if (r < n) {
                            const int q_a = (int)((int64_t)__ldg(rowptr + r) - q0);
                            const int q_e = (int)((int64_t)__ldg(rowptr + r + 1) - q0);
                            for (int q = q_a; q < q_e; q++) sum = __dadd_rn(sum, s_prod[q]);
                            a.z[r] = sum;
                        }
                        s_z[gtid] = sum;
                    }
                } else if (gtid < FU_T) {
                    const int64_t r = r0 + gtid;
                    double sum = 0.0;
                    if (r < n) {
                        for (int64_t q = __ldg(rowptr + r); q < (int64_t)__ldg(rowptr + r + 1); q++)
                            sum = __dadd_rn(sum, __dmul_rn(__ldg(a.val + q), __ldcg(un + __ldg(col + q))));
                        a.z[r] = sum;
                    }
                    s_z[gtid] = sum;
                }
                named_bar(2);
            }
            const int64_t ra = r0 + 2 * lane, rb = ra + 64;
            const double2 ua = ld2_rows(un, ra, n, true, drop), ub = ld2_rows(un, rb, n, true, drop);
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
            for (int g0 = 0; g0 < MAXG; g0 += 4) {  // 4 column groups (8 x 16 B) in flight per lane
                double2 vA[4], vB[4];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const int j = (g0 + c) * FU_WARPS + warp;
                    if (j <= p) {
                        vA[c] = ld2_rows(V + (int64_t)j * ld, ra, n, true, drop);
                        vB[c] = ld2_rows(V + (int64_t)j * ld, rb, n, true, drop);
                    } else {
                        vA[c] = ua;
                        vB[c] = ub;
                    }
                }
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const int g = g0 + c;
                    const int j = g * FU_WARPS + warp;
                    if (j < ncols) {
                        const double2 va = vA[c], vb = vB[c];
                        accu[g] = fma(vb.y, ub.y, fma(vb.x, ub.x, fma(va.y, ua.y, fma(va.x, ua.x, accu[g]))));
                        if (NV2) accz[g] = fma(vb.y, zb.y, fma(vb.x, zb.x, fma(va.y, za.y, fma(va.x, za.x, accz[g]))));
                    }
                }
            }
            named_bar(2);  // s_z / s_prod reused by the next tile
            if (gtid == 0) s_bdone = (int)(k + 1);
        }
    }
    __syncthreads();
    // ================= per-CTA partials, last CTA reduces in CTA order =================
    const int stride = (NV2 && !drain) ? 2 * ncols : ncols;
    if (role == 2) {
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
    }
    __syncthreads();
    for (int i = tid; i < stride; i += FU_CTA_THREADS) a.part[(int64_t)blockIdx.x * stride + i] = s_acc[i];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    final_reduce(a.part, stride, (int)gridDim.x, a.out);
    if (tid == 0) { *a.counter = 0u; a.counter[1] += 1u; }  // [1]: reductions executed
}

static size_t fused_smem(int p) {
    return (size_t)(FU_STAGES * FU_STAGE_D + FU_WARPS * FU_T * 2 + FU_K * FU_THREADS + FU_T + (p + 1) + (p + 2) +
                    2 * (p + 2) + 2) * sizeof(double) + 2 * FU_STAGES * sizeof(uint64_t) + 64;
}

template <int MAXG, bool NV2, bool HA, typename IT, typename PT>
static cudaError_t fused_go(const FusedArgs& a, int grid, cudaStream_t s) {
    auto k = fused_kernel<MAXG, NV2, HA, IT, PT>;
    const size_t smem = fused_smem(a.p);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, FU_CTA_THREADS, smem, s>>>(a);
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
                                                  FU_CTA_THREADS, fused_smem(120));
    if (occ < 1) occ = 1;
    return num_sms;  // one CTA (two warp groups) per SM: bounds the rows in flight
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
