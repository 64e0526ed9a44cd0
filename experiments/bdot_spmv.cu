// bdot_spmv.cu -- SpMV + fused block dot of one Arnoldi iteration in one bulk-copy pipeline:
//
//     z = A u                          (Alg. 3 Step 4: A u_{k-1})
//     [V_p, u]^T [u, z]  -> 2(p+1)      (Alg. 3 Step 4)
//
// Persistent CTA per SM = 1 producer warp + 8 consumer warps, 256-row tiles (CTA c owns
// tiles c, c+G, ...).  Per tile the producer bulk-copies (cp.async.bulk, mbarrier
// expect_tx) into a double-buffered "vector slot": the tile's u rows, its CSR row pointers,
// column indices and values (contiguous ranges of the CSR arrays); then it streams V_p in
// 8-column x 256-row stages (8 x 2 KB copies) through an 8-stage ring.  The consumers
// (a) form the tile's products val * u[col] (u gathered through L2, ghosts from the halo
// buffer), sum each row left to right (the oracle's rounding sequence), write z for the
// update kernel and keep the tile's z in shared memory; (b) multiply every V column of the
// tile against u, z held in registers (warp w owns column 8g+w), one warp reduction per
// column into a per-CTA accumulator only that warp touches.  Stage 2 as in the block dot:
// per-CTA partials, the last CTA sums them in CTA order.  Deterministic, no FP atomics.
//
// Replaces the standalone SpMV kernel + the z round trip and hides the SpMV's dependent
// loads behind the V stream.  Single-rank or multi-rank (ghosts from the halo buffer).
#include <cuda_runtime.h>
#include <stdint.h>

#include "igs_internal.cuh"
#include "ptx_util.cuh"

namespace igs {

#define FULL_MASK 0xffffffffu
constexpr int BS_WARPS = 8;
constexpr int BS_THREADS = (BS_WARPS + 1) * 32;
constexpr int BS_ROWS = 256;
constexpr int BS_RPL = BS_ROWS / 32;               // rows per lane
constexpr int BS_STAGES = 8;
constexpr int BS_STAGE_D = BS_WARPS * BS_ROWS;     // 8 columns x 256 rows = 16 KB
constexpr int BS_NNZ_CAP = BS_ROWS * 8;            // staged nonzeros per tile (mean <= 8/row)
constexpr int BS_VAL_D = BS_NNZ_CAP + 4;           // + alignment slack (16-B bulk copies)
constexpr int BS_COL_I = BS_NNZ_CAP + 8;
constexpr int BS_RP_I = BS_ROWS + 12;             // (multiple of 4 ints: 16-B aligned slots)
static_assert(BS_VAL_D % 2 == 0 && BS_COL_I % 4 == 0 && BS_RP_I % 4 == 0, "bulk-copy slots must stay 16-B aligned");

struct BsArgs {
    int64_t n;
    int p;
    const double* V;
    int64_t ld;
    const double* u;          // V[:, p]
    double* z;                // out: A u
    const int32_t* rowptr;    // int32 CSR (padded by >= 4 entries on the device)
    const int32_t* col;       // local columns (ghost g at n + g); padded by >= 4 entries
    const double* val;        // padded by >= 2 entries
    const double* ghost;      // halo buffer or NULL
    double* part;
    double* out;
    unsigned* counter;
    const int* istate;
};

__device__ __forceinline__ int64_t rdown(int64_t x, int64_t a) { return x & ~(a - 1); }

__global__ void __launch_bounds__(BS_THREADS, 1) bdot_spmv_kernel(BsArgs a) {
    {
        const volatile int* vs = a.istate;
        if (vs && vs[ST_STATUS] != RUNNING) return;
    }
    extern __shared__ __align__(128) double bsm[];
    const int p = a.p;
    const int ncols = p + 1;
    const int stride = 2 * ncols;
    double* ring = bsm;                                   // [STAGES][8][256]
    double* uslot = ring + BS_STAGES * BS_STAGE_D;         // [2][256]
    double* valslot = uslot + 2 * BS_ROWS;                 // [2][VAL_D]
    double* prod = valslot + 2 * BS_VAL_D;                 // [NNZ_CAP]
    double* zs = prod + BS_NNZ_CAP;                        // [256]
    double* acc = zs + BS_ROWS;                            // [2 (p+1)]
    int32_t* colslot = reinterpret_cast<int32_t*>(acc + ((stride + 1) & ~1));  // [2][COL_I]
    int32_t* rpslot = colslot + 2 * BS_COL_I;              // [2][RP_I]
    uint64_t* full = reinterpret_cast<uint64_t*>(rpslot + 2 * BS_RP_I + 8);
    uint64_t* empty = full + BS_STAGES;
    uint64_t* vfull = empty + BS_STAGES;
    uint64_t* vempty = vfull + 2;
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < stride; i += blockDim.x) acc[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < BS_STAGES; s++) { mbar_init(full + s, 1); mbar_init(empty + s, BS_WARPS); }
        for (int s = 0; s < 2; s++) { mbar_init(vfull + s, 1); mbar_init(vempty + s, BS_WARPS); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t n = a.n;
    const int64_t ntiles = (n + BS_ROWS - 1) / BS_ROWS;
    const int ngroups = (p + BS_WARPS - 1) / BS_WARPS;    // V columns only (column p = u)
    const int ncg = (ncols + BS_WARPS - 1) / BS_WARPS;    // consumer groups incl. column p

    if (warp == BS_WARPS) {
        // ================================ producer ================================
        if (lane == 0) {
            const uint64_t stream_pol = l2_policy_evict_first();
            // vector slot of tile k (u rows, CSR row pointers, columns, values): issued one
            // tile ahead of tile k's V stream so the consumers' SpMV never waits for it
            auto issue_slot = [&](int64_t k) {
                const int64_t tile = blockIdx.x + k * gridDim.x;
                const int tb = (int)(k & 1);
                const int64_t row0 = tile * BS_ROWS;
                const int64_t rows = n - row0 < BS_ROWS ? n - row0 : BS_ROWS;
                mbar_wait(vempty + tb, (uint32_t)(((k >> 1) & 1) ^ 1));
                const int64_t q0 = __ldg(a.rowptr + row0), q1 = __ldg(a.rowptr + row0 + rows);
                const int64_t va = rdown(q0, 2), ca = rdown(q0, 4), ra = rdown(row0, 4);
                const uint32_t ub = (uint32_t)(((rows + 1) & ~1LL) * 8);
                const uint32_t vb = (uint32_t)(((q1 - va + 1) & ~1LL) * 8);
                const uint32_t cb = (uint32_t)(((q1 - ca + 3) & ~3LL) * 4);
                const uint32_t rb = (uint32_t)(((row0 + rows + 1 - ra + 3) & ~3LL) * 4);
                mbar_arrive_expect_tx(vfull + tb, ub + vb + cb + rb);
                bulk_g2s(uslot + tb * BS_ROWS, a.u + row0, ub, vfull + tb);
                bulk_g2s_hint(valslot + tb * BS_VAL_D, a.val + va, vb, vfull + tb, stream_pol);
                bulk_g2s_hint(colslot + tb * BS_COL_I, a.col + ca, cb, vfull + tb, stream_pol);
                bulk_g2s(rpslot + tb * BS_RP_I, a.rowptr + ra, rb, vfull + tb);
            };
            const int64_t nk = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            if (nk > 0) issue_slot(0);
            uint32_t it = 0;
            for (int64_t k = 0; k < nk; k++) {
                if (k + 1 < nk) issue_slot(k + 1);
                const int64_t tile = blockIdx.x + k * gridDim.x;
                const int64_t row0 = tile * BS_ROWS;
                const int64_t rows = n - row0 < BS_ROWS ? n - row0 : BS_ROWS;
                const uint32_t ub = (uint32_t)(((rows + 1) & ~1LL) * 8);
                for (int g = 0; g < ngroups; g++, it++) {
                    const int st = it % BS_STAGES;
                    mbar_wait(empty + st, ((it / BS_STAGES) & 1) ^ 1);
                    const int c0 = g * BS_WARPS;
                    const int nc = min(BS_WARPS, p - c0);
                    mbar_arrive_expect_tx(full + st, (uint32_t)nc * ub);
                    for (int c = 0; c < nc; c++)
                        bulk_g2s_hint(ring + (size_t)st * BS_STAGE_D + c * BS_ROWS, a.V + (int64_t)(c0 + c) * a.ld + row0,
                                      ub, full + st, stream_pol);
                }
            }
        }
    } else {
        // ================================ consumers ================================
        const int tid = threadIdx.x;  // 0..255
        uint32_t it = 0;
        int64_t k = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, k++) {
            const int tb = (int)(k & 1);
            const int64_t row0 = tile * BS_ROWS;
            const int64_t rows = n - row0 < BS_ROWS ? n - row0 : BS_ROWS;
            mbar_wait(vfull + tb, (uint32_t)((k >> 1) & 1));
            const int32_t* rps = rpslot + tb * BS_RP_I + (row0 - rdown(row0, 4));
            const int64_t q0 = rps[0], q1 = rps[rows];
            const int cnt = (int)(q1 - q0);
            const double* vs = valslot + tb * BS_VAL_D + (q0 - rdown(q0, 2));
            const int32_t* cs = colslot + tb * BS_COL_I + (q0 - rdown(q0, 4));
            // (a) SpMV of the tile: products in shared memory, rows summed left to right
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int i = tid + j * (BS_WARPS * 32);
                if (i < cnt) {
                    const int64_t c = cs[i];
                    const double xv = (a.ghost && c >= n) ? __ldg(a.ghost + (c - n)) : __ldg(a.u + c);
                    prod[i] = __dmul_rn(vs[i], xv);
                }
            }
            named_barrier(1, BS_WARPS * 32);
            double zrow = 0.0;
            if (tid < rows) {
                const int qa = (int)(rps[tid] - q0), qe = (int)(rps[tid + 1] - q0);
                for (int q = qa; q < qe; q++) zrow = __dadd_rn(zrow, prod[q]);
                a.z[row0 + tid] = zrow;
            }
            zs[tid] = zrow;
            named_barrier(1, BS_WARPS * 32);
            double ur[BS_RPL], zr[BS_RPL];
#pragma unroll
            for (int j = 0; j < BS_RPL; j++) {
                const int r = lane + 32 * j;
                const bool ok = r < rows;
                ur[j] = ok ? uslot[tb * BS_ROWS + r] : 0.0;
                zr[j] = ok ? zs[r] : 0.0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(vempty + tb);
            // (b) block dot against the streamed V columns; column p is u itself
            for (int g = 0; g < ncg; g++) {
                const int c = g * BS_WARPS + warp;
                const bool streamed = g < ngroups;
                const int st = it % BS_STAGES;
                if (streamed) mbar_wait(full + st, (it / BS_STAGES) & 1);
                if (c < ncols) {
                    double su = 0.0, sz = 0.0;
                    if (c < p) {
                        const double* colv = ring + (size_t)st * BS_STAGE_D + warp * BS_ROWS;
#pragma unroll
                        for (int j = 0; j < BS_RPL; j++) {
                            double v = colv[lane + 32 * j];
                            if (lane + 32 * j >= rows) v = 0.0;
                            su = fma(v, ur[j], su);
                            sz = fma(v, zr[j], sz);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < BS_RPL; j++) {
                            su = fma(ur[j], ur[j], su);
                            sz = fma(ur[j], zr[j], sz);
                        }
                    }
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        su += __shfl_xor_sync(FULL_MASK, su, off);
                        sz += __shfl_xor_sync(FULL_MASK, sz, off);
                    }
                    if (lane == 0) {
                        acc[c] += su;
                        acc[ncols + c] += sz;
                    }
                }
                if (streamed) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + st);
                    it++;
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < stride; i += blockDim.x) a.part[(int64_t)blockIdx.x * stride + i] = acc[i];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    final_reduce(a.part, stride, (int)gridDim.x, a.out);  // [V_p^T u, u.u, V_p^T z, u.z]
    if (threadIdx.x == 0) { *a.counter = 0u; a.counter[1] += 1u; }  // [1]: reductions executed
}

static size_t bs_smem(int p) {
    const size_t stride = 2 * (size_t)(p + 1);
    return (size_t)(BS_STAGES * BS_STAGE_D + 2 * BS_ROWS + 2 * BS_VAL_D + BS_NNZ_CAP + BS_ROWS) * 8 +
           ((stride + 1) & ~(size_t)1) * 8 + (size_t)(2 * BS_COL_I + 2 * BS_RP_I + 8) * 4 +
           (2 * BS_STAGES + 4) * 8 + 64;
}

int bdot_spmv_tile_rows() { return BS_ROWS; }
int bdot_spmv_nnz_cap() { return BS_NNZ_CAP; }
bool bdot_spmv_fits(int p) { return bs_smem(p) <= 227 * 1024; }

cudaError_t launch_bdot_spmv(int64_t n, int p, const double* V, int64_t ld, const double* u, double* z,
                             const int32_t* rowptr, const int32_t* col, const double* val,
                             const double* ghost, double* out, double* part, unsigned* counter,
                             int grid, const int* istate, cudaStream_t s) {
    const size_t smem = bs_smem(p);
    const int64_t ntiles = (n + BS_ROWS - 1) / BS_ROWS;
    const int g = (int)(ntiles < grid ? ntiles : grid);
    BsArgs a{n, p, V, ld, u, z, rowptr, col, val, ghost, part, out, counter, istate};
    cudaFuncSetAttribute(bdot_spmv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bdot_spmv_kernel<<<g, BS_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace igs
