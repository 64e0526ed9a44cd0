// fused.cu -- one persistent wavefront kernel per Arnoldi iteration (single GPU, opt-in
// IGS_FUSED=1):
//
//     fused update of iteration p      v_p = (u - V_p r2)/gamma, u' = z/gamma - V_{p+1} r1
//   + SpMV of iteration p+1            z' = A u'
//   + fused block dot of iteration p+1 [V_{p+1}, u']^T [u', z']
//
// The 3-kernel path streams V_p from HBM twice per iteration (update, then block dot one SpMV
// later) -- what the byte model of SURVEY §8(d) counts.  The SpMV's dependence on u' is only a
// band of `reach` rows (one grid plane for the 3D stencil), so tile s can run its SpMV + block
// dot as soon as the update of tiles s-L..s+L is done: phase B re-reads V from the 126 MB L2
// instead of HBM (L2 window ~ (reach + rows in flight) x (p+3) x 8 B, checked by the host).
//
// CTA (one per SM) = 19 warps, every phase a bulk-copy pipeline:
//   warps 0-7   A consumers: update of the CTA's tiles c, c+G, ... (warp w owns column 8g+w of
//               group g; per-row cross-warp sum in shared memory; v_p, u' stored)
//   warp  8     A producer: u, z rows of the tile + V_p in 8-column x 128-row stages
//               (cp.async.bulk, L2 evict_last so phase B finds them)
//   warp  9     publisher: fence + release of the CTA's progress word, off the A critical path
//   warps 10-17 B consumers: SpMV of the tile (u' gathered through L2), z' stored, then the dots
//               of V_0..V_p and u' against u', z' (warp per column, per-CTA accumulators)
//   warp 18     B producer: waits for the neighbourhood's progress words, then bulk-copies the
//               tile's CSR slices and u' rows and re-streams V_0..V_p (L2 evict_first)
// A may lead B by `ahead` own tiles (bounds the L2 window); B waits on the owners' progress.
// Determinism: fixed per-CTA accumulation order, fixed-order stage 2 (final_reduce).
//
// P:n = PAPER.md line n.  Alg. 3 Steps 10-13 and Step 4.
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_internal.cuh"
#include "ptx_util.cuh"

namespace igs {

#define FULL_MASK 0xffffffffu
constexpr int FU_T = 128;                      // rows per tile
constexpr int FU_CW = 8;                       // consumer warps per phase
constexpr int FU_CT = FU_CW * 32;              // consumer threads per phase
constexpr int FU_STAGES = 8;                   // ring depth (each phase)
constexpr int FU_STAGE_D = FU_CW * FU_T;       // 8 columns x 128 rows = 8 KB
constexpr int FU_NNZ_CAP = FU_T * 8;           // staged nonzeros per tile
constexpr int FU_VAL_D = FU_NNZ_CAP + 4;
constexpr int FU_COL_I = FU_NNZ_CAP + 8;
constexpr int FU_RP_I = FU_T + 12;
constexpr int FU_WARPS_ALL = 19;
constexpr int FU_CTA_THREADS = FU_WARPS_ALL * 32;
static_assert(FU_VAL_D % 2 == 0 && FU_COL_I % 4 == 0 && FU_RP_I % 4 == 0, "16-B aligned slots");

__device__ __forceinline__ long long ld_acquire64(const long long* p) {
    long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release64(long long* p, long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t rdown(int64_t x, int64_t a) { return x & ~(a - 1); }

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
    const int32_t* rowptr; // int32 CSR, arrays padded by >= 8 entries
    const int32_t* col;
    const double* val;
    int lag;               // tiles reached by one row's SpMV
    long long* progress;   // per CTA: (epoch << 32) | (last own tile whose phase A finished) + 1
    int epoch;
    double* part;          // [grid * 2 (p+2)]
    double* out;           // dots of iteration p+1
    unsigned* counter;
    const int* istate;
};

template <bool HAS_ALPHA, bool DRAIN>
__global__ void __launch_bounds__(FU_CTA_THREADS, 1) fused_kernel(FusedArgs a) {
    {
        const volatile int* vs = a.istate;
        if (vs[ST_MODE_IT] != a.p || vs[ST_MODE] != 3) return;  // stopped / breakdown
    }
    extern __shared__ __align__(128) double fsm[];
    const int p = a.p;
    const int ncols = p + 2;                           // V_0..V_p and u' itself
    const int stride = DRAIN ? ncols : 2 * ncols;
    double* ringA = fsm;                               // [STAGES][8][128]
    double* ringB = ringA + FU_STAGES * FU_STAGE_D;    // [STAGES][8][128]
    double* aslot = ringB + FU_STAGES * FU_STAGE_D;    // [2][u | z][128]
    double* s_red = aslot + 4 * FU_T;                  // [8][128][2]
    double* bval = s_red + FU_CW * FU_T * 2;           // [2][VAL_D]
    double* bu = bval + 2 * FU_VAL_D;                  // [2][128] u' rows
    double* prod = bu + 2 * FU_T;                      // [NNZ_CAP]
    double* zs = prod + FU_NNZ_CAP;                    // [128]
    double* s_alpha = zs + FU_T;                       // [p+1]
    double* s_beta = s_alpha + (p + 2);                // [p+2]
    double* acc = s_beta + (p + 2);                    // [2 ncols]
    int32_t* bcol = reinterpret_cast<int32_t*>(acc + 2 * ncols + 2);   // [2][COL_I]
    int32_t* brp = bcol + 2 * FU_COL_I;                                 // [2][RP_I]
    uint64_t* bar = reinterpret_cast<uint64_t*>(brp + 2 * FU_RP_I + 8);
    uint64_t* fullA = bar;                      // [STAGES]
    uint64_t* emptyA = fullA + FU_STAGES;       // [STAGES]
    uint64_t* fullB = emptyA + FU_STAGES;       // [STAGES]
    uint64_t* emptyB = fullB + FU_STAGES;       // [STAGES]
    uint64_t* afull = emptyB + FU_STAGES;       // [2] A vector slot
    uint64_t* aempty = afull + 2;               // [2]
    uint64_t* bfull = aempty + 2;               // [2] B vector slot
    uint64_t* bempty = bfull + 2;               // [2]
    __shared__ bool s_last;
    __shared__ volatile int s_adone, s_bdone;   // own tiles finished by phase A / phase B
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int j = tid; j < p; j += FU_CTA_THREADS) s_alpha[j] = HAS_ALPHA ? a.alpha[j] : 0.0;
    for (int j = tid; j <= p; j += FU_CTA_THREADS) s_beta[j] = a.beta[j];
    for (int i = tid; i < 2 * ncols; i += FU_CTA_THREADS) acc[i] = 0.0;
    if (tid == 0) {
        s_adone = 0;
        s_bdone = 0;
        for (int s = 0; s < FU_STAGES; s++) {
            mbar_init(fullA + s, 1); mbar_init(emptyA + s, FU_CW);
            mbar_init(fullB + s, 1); mbar_init(emptyB + s, FU_CW);
        }
        for (int s = 0; s < 2; s++) {
            mbar_init(afull + s, 1); mbar_init(aempty + s, FU_CW);
            mbar_init(bfull + s, 1); mbar_init(bempty + s, FU_CW);
        }
        mbar_fence_init();
    }
    const double gamma = *a.gamma;
    __syncthreads();

    const int64_t n = a.n, ld = a.ld;
    const double* __restrict__ V = a.V;
    double* u = const_cast<double*>(V) + (int64_t)p * ld;         // pending -> v_p in place
    double* un = const_cast<double*>(V) + (int64_t)(p + 1) * ld;  // u'
    const int64_t ntiles = (n + FU_T - 1) / FU_T;
    const int64_t G = gridDim.x;
    const int64_t nown = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
    const int L = a.lag;
    const int ahead = (int)((L + G - 1) / G) + 2;
    const int ngA = (p + FU_CW - 1) / FU_CW;          // phase A streams V_0..V_{p-1}
    const int ngB = (p + 1 + FU_CW - 1) / FU_CW;      // phase B streams V_0..V_p
    const int ncgB = (ncols + FU_CW - 1) / FU_CW;     // + u' itself

    if (warp == 8) {
        // =========================== A producer ===========================
        if (lane == 0) {
            const uint64_t keep = l2_policy_evict_last();
            uint32_t it = 0;
            for (int64_t k = 0; k < nown; k++) {
                while (s_bdone < k - ahead) __nanosleep(128);
                const int tb = (int)(k & 1);
                const int64_t r0 = (blockIdx.x + k * G) * FU_T;
                const int64_t rows = n - r0 < FU_T ? n - r0 : FU_T;
                const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * 8);
                mbar_wait(aempty + tb, (uint32_t)(((k >> 1) & 1) ^ 1));
                mbar_arrive_expect_tx(afull + tb, 2 * bytes);
                bulk_g2s(aslot + (2 * tb) * FU_T, u + r0, bytes, afull + tb);
                bulk_g2s(aslot + (2 * tb + 1) * FU_T, a.z + r0, bytes, afull + tb);
                for (int g = 0; g < ngA; g++, it++) {
                    const int st = it % FU_STAGES;
                    mbar_wait(emptyA + st, ((it / FU_STAGES) & 1) ^ 1);
                    const int c0 = g * FU_CW, nc = min(FU_CW, p - c0);
                    mbar_arrive_expect_tx(fullA + st, (uint32_t)nc * bytes);
                    for (int c = 0; c < nc; c++)
                        bulk_g2s_hint(ringA + (size_t)st * FU_STAGE_D + c * FU_T, V + (int64_t)(c0 + c) * ld + r0,
                                      bytes, fullA + st, keep);
                }
            }
        }
    } else if (warp == 9) {
        // =========================== publisher ===========================
        if (lane == 0) {
            for (int64_t k = 0; k < nown; k++) {
                while (s_adone < k + 1) __nanosleep(64);
                __threadfence();  // cumulative: the A consumers' stores precede the release
                st_release64(a.progress + blockIdx.x,
                             ((long long)a.epoch << 32) | (long long)(blockIdx.x + k * G + 1));
            }
        }
    } else if (warp < 8) {
        // =========================== A consumers ===========================
        uint32_t it = 0;
        for (int64_t k = 0; k < nown; k++) {
            const int tb = (int)(k & 1);
            const int64_t r0 = (blockIdx.x + k * G) * FU_T;
            const int64_t rows = n - r0 < FU_T ? n - r0 : FU_T;
            double t1[4] = {0.0, 0.0, 0.0, 0.0}, t2[4] = {0.0, 0.0, 0.0, 0.0};
            for (int g = 0; g < ngA; g++, it++) {
                const int st = it % FU_STAGES;
                const int c = g * FU_CW + warp;
                mbar_wait(fullA + st, (it / FU_STAGES) & 1);
                if (c < p) {
                    const double* cs = ringA + (size_t)st * FU_STAGE_D + warp * FU_T;
                    const double al = s_alpha[c], be = s_beta[c];
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const double v = (lane + 32 * i < rows) ? cs[lane + 32 * i] : 0.0;
                        if (HAS_ALPHA) t1[i] = fma(v, al, t1[i]);
                        t2[i] = fma(v, be, t2[i]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(emptyA + st);
            }
            double* rw = s_red + warp * FU_T * 2;
#pragma unroll
            for (int i = 0; i < 4; i++) { rw[2 * (lane + 32 * i)] = t1[i]; rw[2 * (lane + 32 * i) + 1] = t2[i]; }
            mbar_wait(afull + tb, (uint32_t)((k >> 1) & 1));
            named_barrier(1, FU_CT);
            if (tid < FU_T && tid < rows) {
                double T1 = 0.0, T2 = 0.0;
#pragma unroll
                for (int ww = 0; ww < FU_CW; ww++) {
                    T1 += s_red[(ww * FU_T + tid) * 2];
                    T2 += s_red[(ww * FU_T + tid) * 2 + 1];
                }
                const double uu = aslot[(2 * tb) * FU_T + tid], zz = aslot[(2 * tb + 1) * FU_T + tid];
                const double v = (HAS_ALPHA ? uu - T1 : uu) / gamma;
                u[r0 + tid] = v;
                un[r0 + tid] = zz / gamma - fma(v, s_beta[p], T2);
            }
            named_barrier(1, FU_CT);  // s_red and the slot are free again; stores issued
            if (tid == 0) {
                for (int w = 0; w < FU_CW; w++) mbar_arrive(aempty + tb);
                __threadfence_block();
                s_adone = (int)(k + 1);
            }
        }
    } else if (warp == 18) {
        // =========================== B producer ===========================
        const uint64_t drop = l2_policy_evict_first();
        uint32_t it = 0;
        for (int64_t k = 0; k < nown; k++) {
            const int tb = (int)(k & 1);
            const int64_t s = blockIdx.x + k * G;
            const int64_t r0 = s * FU_T;
            const int64_t rows = n - r0 < FU_T ? n - r0 : FU_T;
            // neighbourhood [s-L, s+L]: the owner of tile t is t % G and finishes its tiles in order
            const int64_t t0 = s - L > 0 ? s - L : 0;
            const int64_t t1 = s + L < ntiles - 1 ? s + L : ntiles - 1;
            const int64_t span = t1 - t0 + 1;
            const int64_t nchk = span < G ? span : G;
            for (int64_t q = lane; q < nchk; q += 32) {
                const int64_t owner = (t1 - q) % G;
                const long long need = ((long long)a.epoch << 32) | (long long)(t1 - q + 1);
                while (ld_acquire64(a.progress + owner) < need) __nanosleep(64);
            }
            __syncwarp();
            if (lane == 0) {
                const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * 8);
                mbar_wait(bempty + tb, (uint32_t)(((k >> 1) & 1) ^ 1));
                uint32_t tx = bytes;
                int64_t q0 = 0, q1 = 0;
                if (!DRAIN) {
                    q0 = __ldg(a.rowptr + r0);
                    q1 = __ldg(a.rowptr + r0 + rows);
                    tx += (uint32_t)(((q1 - rdown(q0, 2) + 1) & ~1LL) * 8) + (uint32_t)(((q1 - rdown(q0, 4) + 3) & ~3LL) * 4) +
                          (uint32_t)(((r0 + rows + 1 - rdown(r0, 4) + 3) & ~3LL) * 4);
                }
                mbar_arrive_expect_tx(bfull + tb, tx);
                bulk_g2s(bu + tb * FU_T, un + r0, bytes, bfull + tb);
                if (!DRAIN) {
                    bulk_g2s_hint(bval + tb * FU_VAL_D, a.val + rdown(q0, 2), (uint32_t)(((q1 - rdown(q0, 2) + 1) & ~1LL) * 8), bfull + tb, drop);
                    bulk_g2s_hint(bcol + tb * FU_COL_I, a.col + rdown(q0, 4), (uint32_t)(((q1 - rdown(q0, 4) + 3) & ~3LL) * 4), bfull + tb, drop);
                    bulk_g2s(brp + tb * FU_RP_I, a.rowptr + rdown(r0, 4), (uint32_t)(((r0 + rows + 1 - rdown(r0, 4) + 3) & ~3LL) * 4), bfull + tb);
                }
                for (int g = 0; g < ngB; g++, it++) {
                    const int st = it % FU_STAGES;
                    mbar_wait(emptyB + st, ((it / FU_STAGES) & 1) ^ 1);
                    const int c0 = g * FU_CW, nc = min(FU_CW, p + 1 - c0);
                    mbar_arrive_expect_tx(fullB + st, (uint32_t)nc * bytes);
                    for (int c = 0; c < nc; c++)
                        bulk_g2s_hint(ringB + (size_t)st * FU_STAGE_D + c * FU_T, V + (int64_t)(c0 + c) * ld + r0,
                                      bytes, fullB + st, drop);
                }
            }
        }
    } else {
        // =========================== B consumers (warps 10-17) ===========================
        const int bw = warp - 10, btid = tid - 10 * 32;
        uint32_t it = 0;
        for (int64_t k = 0; k < nown; k++) {
            const int tb = (int)(k & 1);
            const int64_t r0 = (blockIdx.x + k * G) * FU_T;
            const int64_t rows = n - r0 < FU_T ? n - r0 : FU_T;
            mbar_wait(bfull + tb, (uint32_t)((k >> 1) & 1));
            if (!DRAIN) {
                const int32_t* rps = brp + tb * FU_RP_I + (r0 - rdown(r0, 4));
                const int64_t q0 = rps[0], q1 = rps[rows];
                const int cnt = (int)(q1 - q0);
                const double* vs = bval + tb * FU_VAL_D + (q0 - rdown(q0, 2));
                const int32_t* cs = bcol + tb * FU_COL_I + (q0 - rdown(q0, 4));
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int i = btid + j * FU_CT;
                    if (i < cnt) prod[i] = __dmul_rn(vs[i], __ldcg(un + cs[i]));
                }
                named_barrier(2, FU_CT);
                double zr = 0.0;
                if (btid < rows) {
                    const int qa = (int)(rps[btid] - q0), qe = (int)(rps[btid + 1] - q0);
                    for (int q = qa; q < qe; q++) zr = __dadd_rn(zr, prod[q]);
                    a.z[r0 + btid] = zr;
                }
                if (btid < FU_T) zs[btid] = zr;
                named_barrier(2, FU_CT);
            }
            double ur[4], zr4[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const bool ok = lane + 32 * i < rows;
                ur[i] = ok ? bu[tb * FU_T + lane + 32 * i] : 0.0;
                zr4[i] = (!DRAIN && ok) ? zs[lane + 32 * i] : 0.0;
            }
            for (int g = 0; g < ncgB; g++) {
                const int c = g * FU_CW + bw;
                const bool streamed = g < ngB;
                const int st = it % FU_STAGES;
                if (streamed) mbar_wait(fullB + st, (it / FU_STAGES) & 1);
                if (c < ncols) {
                    double su = 0.0, sz = 0.0;
                    if (c <= p) {
                        const double* cv = ringB + (size_t)st * FU_STAGE_D + bw * FU_T;
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            const double v = (lane + 32 * i < rows) ? cv[lane + 32 * i] : 0.0;
                            su = fma(v, ur[i], su);
                            sz = fma(v, zr4[i], sz);
                        }
                    } else {  // u' itself
#pragma unroll
                        for (int i = 0; i < 4; i++) { su = fma(ur[i], ur[i], su); sz = fma(ur[i], zr4[i], sz); }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        su += __shfl_xor_sync(FULL_MASK, su, off);
                        sz += __shfl_xor_sync(FULL_MASK, sz, off);
                    }
                    if (lane == 0) {
                        acc[c] += su;
                        if (!DRAIN) acc[ncols + c] += sz;
                    }
                }
                if (streamed) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(emptyB + st);
                    it++;
                }
            }
            named_barrier(2, FU_CT);  // zs / prod reuse
            if (btid == 0) {
                for (int w = 0; w < FU_CW; w++) mbar_arrive(bempty + tb);
                s_bdone = (int)(k + 1);
            }
        }
    }
    __syncthreads();
    // ================= per-CTA partials, last CTA reduces in fixed order =================
    for (int i = tid; i < stride; i += FU_CTA_THREADS) a.part[(int64_t)blockIdx.x * stride + i] = acc[i];
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    final_reduce(a.part, stride, (int)gridDim.x, a.out);  // [V^T u', u'.u', V^T z', u'.z']
    if (tid == 0) { *a.counter = 0u; a.counter[1] += 1u; }
}

static size_t fused_smem(int p) {
    const size_t nd = 2 * FU_STAGES * FU_STAGE_D + 4 * FU_T + FU_CW * FU_T * 2 + 2 * FU_VAL_D + 2 * FU_T +
                      FU_NNZ_CAP + FU_T + (p + 2) + (p + 2) + 2 * (p + 2) + 2;
    return nd * 8 + (size_t)(2 * FU_COL_I + 2 * FU_RP_I + 8) * 4 + (4 * FU_STAGES + 8) * 8 + 128;
}

int fused_max_cols() {
    for (int p = 1; p < 4096; p++)
        if (fused_smem(p) > 227 * 1024) return p + 1;
    return 4096;
}
int fused_tile_rows() { return FU_T; }
int fused_nnz_cap() { return FU_NNZ_CAP; }
int fused_grid(int num_sms) { return num_sms; }  // one CTA (19 warps) per SM

cudaError_t launch_fused(int64_t n, int p, int m, const double* V, int64_t ld, double* z,
                         const double* alpha, const double* beta, const double* gamma_dev,
                         const SpmvArgs& A, int lag, long long* progress, int epoch, double* part,
                         double* out, unsigned* counter, const int* istate, int grid,
                         cudaStream_t s) {
    if (A.idx64 || A.ptr64) return cudaErrorNotSupported;
    FusedArgs a{n, p, m, V, ld, z, alpha, beta, gamma_dev, static_cast<const int32_t*>(A.rowptr),
                static_cast<const int32_t*>(A.col), A.val, lag, progress, epoch, part, out, counter, istate};
    const size_t smem = fused_smem(p);
    const bool drain = (p + 1 == m);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, FU_CTA_THREADS, smem, s>>>(a);
    };
    if (alpha) { if (drain) go(fused_kernel<true, true>); else go(fused_kernel<true, false>); }
    else { if (drain) go(fused_kernel<false, true>); else go(fused_kernel<false, false>); }
    return cudaGetLastError();
}

}  // namespace igs
