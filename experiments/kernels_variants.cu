// experiments/kernels_variants.cu -- measured-slower variants removed from libigs.so.
//
// NOT BUILT.  Kept as source for the negative results in DESIGN.md §7.4 (numbers there):
//   bdot_tmap_kernel    block dot with 2D TMA tensor copies (box 256 x 8): 4.7 vs 6.3 TB/s on c4
//   bdot_stream_kernel  block dot streaming 512-row warp ranges through registers: no gain
//   update_tma_kernel   fused update with V_p bulk-copied into shared memory: 6.5 vs 6.9 TB/s
// They were written against the round-1 kernels.cu (ptx_util.cuh helpers, bfly8, running(),
// BT_* constants) and would need those definitions to compile again.
// ------------------------------------------------------------------------------------
// K2 (TMA tensor variant, the default): same structure as bdot_tma_kernel, but V is
// streamed with 2D tensor copies -- one cp.async.bulk.tensor instruction per 8-column x
// 256-row box (16 KB) -- because a single producer thread issuing 1D bulk copies tops out at
// a few copies per microsecond (1-4 KB copies measured at 1.7-7 TB/s).  Rows past n and
// columns past the map come back zero-filled.  12-stage ring (192 KB) per SM.
// ------------------------------------------------------------------------------------
constexpr int TM_ROWS = 256;
constexpr int TM_RPL = TM_ROWS / 32;
constexpr int TM_STAGES = 12;
constexpr int TM_STAGE_D = BT_CONS_WARPS * TM_ROWS;  // 8 columns x 256 rows = 16 KB

template <int NV>
__global__ void __launch_bounds__(BT_THREADS, 1)
    bdot_tmap_kernel(const __grid_constant__ CUtensorMap tmV, int64_t n, int p,
                     const double* __restrict__ u, const double* __restrict__ z,
                     double* __restrict__ part, double* __restrict__ out, unsigned* counter,
                     const int* istate) {
    if (!running(istate)) return;
    extern __shared__ __align__(128) double smem_tm[];
    double* ring = smem_tm;                                        // [STAGES][8][256]
    double* uzslot = ring + TM_STAGES * TM_STAGE_D;                // [2 tiles][u | z][256]
    double* acc = uzslot + 4 * TM_ROWS;                            // [NV*(p+1)]
    const int ncols = p + 1;
    const int stride = NV * ncols;
    uint64_t* full = reinterpret_cast<uint64_t*>(acc + ((stride + 1) & ~1));
    uint64_t* empty = full + TM_STAGES;
    uint64_t* uzfull = empty + TM_STAGES;
    uint64_t* uzempty = uzfull + 2;
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < stride; i += blockDim.x) acc[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < TM_STAGES; s++) { mbar_init(full + s, 1); mbar_init(empty + s, BT_CONS_WARPS); }
        for (int s = 0; s < 2; s++) { mbar_init(uzfull + s, 1); mbar_init(uzempty + s, BT_CONS_WARPS); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t ntiles = (n + TM_ROWS - 1) / TM_ROWS;
    const int ngroups = (ncols + BT_CONS_WARPS - 1) / BT_CONS_WARPS;
    const int nstream = (p + BT_CONS_WARPS - 1) / BT_CONS_WARPS;  // groups holding V columns
    const int64_t nk = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp == BT_CONS_WARPS) {
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_first();
            auto issue_uz = [&](int64_t k) {
                const int tb = (int)(k & 1);
                const int64_t row0 = (blockIdx.x + k * gridDim.x) * TM_ROWS;
                mbar_wait(uzempty + tb, (uint32_t)(((k >> 1) & 1) ^ 1));
                if (row0 + TM_ROWS <= n) {
                    const uint32_t b = TM_ROWS * sizeof(double);
                    mbar_arrive_expect_tx(uzfull + tb, (NV == 2 ? 2 : 1) * b);
                    bulk_g2s(uzslot + (2 * tb) * TM_ROWS, u + row0, b, uzfull + tb);
                    if (NV == 2) bulk_g2s(uzslot + (2 * tb + 1) * TM_ROWS, z + row0, b, uzfull + tb);
                } else {
                    mbar_arrive(uzfull + tb);
                }
            };
            if (nk > 0) issue_uz(0);
            uint32_t it = 0;
            for (int64_t k = 0; k < nk; k++) {
                if (k + 1 < nk) issue_uz(k + 1);
                const int row0 = (int)((blockIdx.x + k * gridDim.x) * TM_ROWS);
                for (int g = 0; g < nstream; g++, it++) {
                    const int st = it % TM_STAGES;
                    mbar_wait(empty + st, ((it / TM_STAGES) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + st, TM_STAGE_D * sizeof(double));
                    tma_load_2d(ring + (size_t)st * TM_STAGE_D, &tmV, row0, g * BT_CONS_WARPS, full + st, pol);
                }
            }
        }
    } else {
        uint32_t it = 0;
        for (int64_t kt = 0; kt < nk; kt++) {
            const int64_t row0 = (blockIdx.x + kt * gridDim.x) * TM_ROWS;
            const bool full_tile = row0 + TM_ROWS <= n;
            const int tb = (int)(kt & 1);
            double ur[TM_RPL], zr[TM_RPL];
            mbar_wait(uzfull + tb, (uint32_t)((kt >> 1) & 1));
            if (full_tile) {
                const double* us = uzslot + (2 * tb) * TM_ROWS;
                const double* zs = uzslot + (2 * tb + 1) * TM_ROWS;
#pragma unroll
                for (int k = 0; k < TM_RPL; k++) {
                    ur[k] = us[lane + 32 * k];
                    zr[k] = NV == 2 ? zs[lane + 32 * k] : 0.0;
                }
            } else {
#pragma unroll
                for (int k = 0; k < TM_RPL; k++) {
                    const int64_t r = row0 + lane + 32 * k;
                    const bool ok = r < n;
                    ur[k] = ok ? __ldg(u + r) : 0.0;
                    zr[k] = (NV == 2 && ok) ? __ldg(z + r) : 0.0;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(uzempty + tb);
            for (int g = 0; g < ngroups; g++) {
                const int c = g * BT_CONS_WARPS + warp;
                const bool streamed = g < nstream;
                const int st = it % TM_STAGES;
                if (streamed) mbar_wait(full + st, (it / TM_STAGES) & 1);
                if (c < ncols) {
                    double su = 0.0, sz = 0.0;
                    if (c < p) {
                        const double* col = ring + (size_t)st * TM_STAGE_D + warp * TM_ROWS;
#pragma unroll
                        for (int k = 0; k < TM_RPL; k++) {
                            const double v = col[lane + 32 * k];   // rows >= n are zero-filled
                            su = fma(v, ur[k], su);
                            if (NV == 2) sz = fma(v, zr[k], sz);
                        }
                    } else {  // column p is u itself
#pragma unroll
                        for (int k = 0; k < TM_RPL; k++) {
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
                        acc[c] += su;
                        if (NV == 2) acc[ncols + c] += sz;
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
    for (int i = threadIdx.x; i < stride; i += blockDim.x) part[(int64_t)blockIdx.x * stride + i] = acc[i];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    final_reduce(part, stride, (int)gridDim.x, out);  // [V_p^T u, u.u, V_p^T z, u.z]
    if (threadIdx.x == 0) { *counter = 0u; counter[1] += 1u; }
}

static size_t bdot_tmap_smem(int p, int nv) {
    const size_t stride = (size_t)nv * (p + 1);
    return (size_t)(TM_STAGES * TM_STAGE_D + 4 * TM_ROWS) * sizeof(double) +
           ((stride + 1) & ~(size_t)1) * sizeof(double) + (2 * TM_STAGES + 4) * sizeof(uint64_t);
}

// ------------------------------------------------------------------------------------
// K2 (streaming variant): each warp owns a 512-row sub-range (8 chunks of 64 rows; a lane
// owns rows 2l, 2l+1 of every chunk) and walks ALL column groups over it, accumulating 8
// column partials per vector in registers across the 8 chunks; the butterfly reduction runs
// once per (512 rows x 8 columns) instead of once per 128 rows.  Loads of the next chunk are
// in flight while the current one is multiplied (16 x 16 B per lane).  u, z of the warp's
// rows are read from shared memory.  Per-warp shared accumulators, fixed-order stage 2.
// ------------------------------------------------------------------------------------
constexpr int BS2_WARPS = 8;
constexpr int BS2_CHUNKS = 8;                      // 64-row chunks per warp
constexpr int BS2_ROWS_W = 64 * BS2_CHUNKS;        // 512 rows per warp
constexpr int BS2_TILE = BS2_WARPS * BS2_ROWS_W;   // 4096 rows per CTA tile

template <int NV>
__global__ void __launch_bounds__(BS2_WARPS * 32, 2)
    bdot_stream_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                       const double* __restrict__ u, const double* __restrict__ z,
                       double* __restrict__ part, double* __restrict__ out, unsigned* counter,
                       const int* istate) {
    if (!running(istate)) return;
    extern __shared__ __align__(16) double sst[];
    const int ncols = p + 1;
    const int stride = NV * ncols;
    double* suz = sst;                                   // [NV][4096]
    double* sacc = sst + NV * BS2_TILE;                  // [8 warps][stride]
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* acc = sacc + warp * stride;
    for (int i = lane; i < stride; i += 32) acc[i] = 0.0;
    const int64_t ntiles = (n + BS2_TILE - 1) / BS2_TILE;
    const int ngroups = (ncols + 7) / 8;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t t0 = tile * BS2_TILE;
        __syncthreads();
        for (int i = threadIdx.x; i < BS2_TILE; i += blockDim.x) {
            const int64_t r = t0 + i;
            suz[i] = r < n ? __ldg(u + r) : 0.0;
            if (NV == 2) suz[BS2_TILE + i] = r < n ? __ldg(z + r) : 0.0;
        }
        __syncthreads();
        const int64_t w0 = t0 + warp * BS2_ROWS_W;     // this warp's 512 rows
        const bool fullw = w0 + BS2_ROWS_W <= n;
        const double* us = suz + warp * BS2_ROWS_W;
        const double* zs = suz + BS2_TILE + warp * BS2_ROWS_W;
        for (int g = 0; g < ngroups; g++) {
            const double* cp[8];
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int j = min(g * 8 + c, ncols - 1);
                cp[c] = (j < p) ? V + (int64_t)j * ld : u;
            }
            double au[8], az[8];
#pragma unroll
            for (int c = 0; c < 8; c++) { au[c] = 0.0; az[c] = 0.0; }
#pragma unroll 2
            for (int ch = 0; ch < BS2_CHUNKS; ch++) {
                const int64_t r = w0 + ch * 64 + 2 * lane;
                double2 v[8];
#pragma unroll
                for (int c = 0; c < 8; c++) v[c] = fullw ? __ldg(reinterpret_cast<const double2*>(cp[c] + r)) : ld2_guard(cp[c], r, n);
                const double2 uu = *reinterpret_cast<const double2*>(us + ch * 64 + 2 * lane);
                double2 zz = make_double2(0.0, 0.0);
                if (NV == 2) zz = *reinterpret_cast<const double2*>(zs + ch * 64 + 2 * lane);
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    au[c] = fma(v[c].y, uu.y, fma(v[c].x, uu.x, au[c]));
                    if (NV == 2) az[c] = fma(v[c].y, zz.y, fma(v[c].x, zz.x, az[c]));
                }
            }
#pragma unroll
            for (int c = 0; c < 8; c++)
                if (g * 8 + c >= ncols) { au[c] = 0.0; az[c] = 0.0; }
            const double su = bfly8(au, lane);
            double sz = 0.0;
            if (NV == 2) sz = bfly8(az, lane);
            const int j = g * 8 + (lane >> 2);
            if ((lane & 3) == 0 && j < ncols) {
                acc[j] += su;
                if (NV == 2) acc[ncols + j] += sz;
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < stride; i += blockDim.x) {
        double sacc2 = 0.0;
#pragma unroll
        for (int w = 0; w < BS2_WARPS; w++) sacc2 += sacc[w * stride + i];
        part[(int64_t)blockIdx.x * stride + i] = sacc2;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    final_reduce(part, stride, (int)gridDim.x, out);  // [V_p^T u, u.u, V_p^T z, u.z]
    if (threadIdx.x == 0) { *counter = 0u; counter[1] += 1u; }
}


// ------------------------------------------------------------------------------------
// K5 (sm_100a pipeline): the same fused update with V_p streamed by the bulk-copy engine,
// as in bdot_tma_kernel: persistent CTA per SM = 8 consumer warps + 1 producer warp, 512-row
// tiles, 8 columns x 512 rows per stage, 6-stage ring.  Consumer warp w owns rows
// 64w + 2l, 64w + 2l + 1 of the tile (one 16-B shared load per column) and accumulates
// t1 = V alpha, t2 = V beta over the columns in ascending order -- the same FMA sequence as
// update_kernel, so the results are bitwise identical; no cross-lane reduction exists.  u
// and z of the tile are fetched into registers when the tile starts and used in the
// epilogue.  Opt-in (IGS_UPDATE_TMA=1): in the c4 bench it streams 6.5 TB/s against the
// register kernel's 6.9 TB/s.
// ------------------------------------------------------------------------------------
template <bool HAS_ALPHA>
__global__ void __launch_bounds__(BT_THREADS, 1)
    update_tma_kernel(int64_t n, int p, const double* __restrict__ V, int64_t ld,
                      const double* u, const double* __restrict__ z,
                      const double* __restrict__ alpha, const double* __restrict__ beta,
                      const double* __restrict__ gamma_dev, double* v_out, double* u_next,
                      const int* istate, int it, int default_mode, const double* __restrict__ zdiv_dev) {
    int mode = default_mode;
    if (istate) {
        const volatile int* vs = istate;
        mode = (vs[ST_MODE_IT] == it) ? vs[ST_MODE] : 0;
        mode &= default_mode;
    }
    if (mode == 0) return;
    const bool want_next = (mode & 2) != 0;
    extern __shared__ __align__(128) double smem_ut[];
    double* ring = smem_ut;                                  // [STAGES][8][512]
    double* sa = ring + BT_STAGES * BT_STAGE_DOUBLES;        // alpha [p]
    double* sb = sa + ((p + 1) & ~1);                        // beta [p+1]
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + ((p + 2) & ~1));
    uint64_t* empty = full + BT_STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (HAS_ALPHA)
        for (int j = threadIdx.x; j < p; j += blockDim.x) sa[j] = alpha[j];
    if (want_next)
        for (int j = threadIdx.x; j <= p; j += blockDim.x) sb[j] = beta[j];
    if (threadIdx.x == 0) {
        for (int st = 0; st < BT_STAGES; st++) { mbar_init(full + st, 1); mbar_init(empty + st, BT_CONS_WARPS); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t ntiles = (n + BT_ROWS - 1) / BT_ROWS;
    const int ngroups = (p + BT_CONS_WARPS - 1) / BT_CONS_WARPS;
    const int64_t nk = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp == BT_CONS_WARPS) {
        if (lane == 0) {
            uint32_t itg = 0;
            for (int64_t k = 0; k < nk; k++) {
                const int64_t row0 = (blockIdx.x + k * gridDim.x) * BT_ROWS;
                const int64_t rows = (n - row0 < BT_ROWS) ? n - row0 : BT_ROWS;
                const uint32_t bytes = (uint32_t)(((rows + 1) & ~1LL) * sizeof(double));
                for (int g = 0; g < ngroups; g++, itg++) {
                    const int st = itg % BT_STAGES;
                    mbar_wait(empty + st, ((itg / BT_STAGES) & 1) ^ 1);
                    const int c0 = g * BT_CONS_WARPS;
                    const int nc = min(BT_CONS_WARPS, p - c0);
                    mbar_arrive_expect_tx(full + st, (uint32_t)nc * bytes);
                    for (int c = 0; c < nc; c++)
                        bulk_g2s(ring + (size_t)st * BT_STAGE_DOUBLES + c * BT_ROWS,
                                 V + (int64_t)(c0 + c) * ld + row0, bytes, full + st);
                }
            }
        }
        return;
    }
    const double gamma = *gamma_dev;
    const double zdiv = zdiv_dev ? *zdiv_dev : gamma;
    const int rl = 64 * warp + 2 * lane;  // this lane's two rows within the tile
    uint32_t itg = 0;
    for (int64_t kt = 0; kt < nk; kt++) {
        const int64_t row0 = (blockIdx.x + kt * gridDim.x) * BT_ROWS;
        const int64_t r = row0 + rl;
        const bool pair = r + 1 < n;
        // epilogue operands, in flight while the tile streams
        const double2 uu = ld2_guard(u, r, n);
        const double2 zz = want_next ? ld2_guard(z, r, n) : make_double2(0.0, 0.0);
        double2 t1 = make_double2(0.0, 0.0), t2 = make_double2(0.0, 0.0);
        for (int g = 0; g < ngroups; g++, itg++) {
            const int st = itg % BT_STAGES;
            mbar_wait(full + st, (itg / BT_STAGES) & 1);
            const int c0 = g * BT_CONS_WARPS;
            const int nc = min(BT_CONS_WARPS, p - c0);
            const double* stg = ring + (size_t)st * BT_STAGE_DOUBLES + rl;
#pragma unroll
            for (int c = 0; c < BT_CONS_WARPS; c++) {
                if (c < nc) {
                    const double2 v = *reinterpret_cast<const double2*>(stg + c * BT_ROWS);
                    if (HAS_ALPHA) { t1.x = fma(v.x, sa[c0 + c], t1.x); t1.y = fma(v.y, sa[c0 + c], t1.y); }
                    if (want_next) { t2.x = fma(v.x, sb[c0 + c], t2.x); t2.y = fma(v.y, sb[c0 + c], t2.y); }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);
        }
        if (r < n) {
            double2 w = uu;
            if (HAS_ALPHA) { w.x = uu.x - t1.x; w.y = uu.y - t1.y; }
            double2 v;
            v.x = w.x / gamma;
            v.y = w.y / gamma;
            if (want_next) {
                const double bp = sb[p];
                u_next[r] = zz.x / zdiv - fma(v.x, bp, t2.x);
                if (pair) u_next[r + 1] = zz.y / zdiv - fma(v.y, bp, t2.y);
            }
            if (mode & 1) {
                v_out[r] = v.x;
                if (pair) v_out[r + 1] = v.y;
            }
        }
    }
}

static size_t update_tma_smem(int p) {
    return (size_t)(BT_STAGES * BT_STAGE_DOUBLES + ((p + 1) & ~1) + ((p + 2) & ~1)) * sizeof(double) +
           2 * BT_STAGES * sizeof(uint64_t);
}

