// experiments/spmv_sell_pipe.cu -- NOT BUILT.  The all-diagonal SELL-32 SpMV with the matrix
// streamed by the bulk-copy engine (round 2, cut from csrc/kernels.cu at the commit after
// "SELL diagonal slices stored by list position"; uses its SellDev / SpmvArgs / ptx_util.cuh).
// Bitwise equal to the oracle's row loop in the GPU tests (65 passed with it as the default).
// Measured on c4, one B200, bench step of 100 SpMVs: 24.9 ms (16 consumer warps x 3 stages x
// 2 CTAs/SM; 8 x 4 x 3: 31.4 ms) against 23.3 ms for one short-lived warp per slice and
// 20.7 ms for the resident warps walking slices that replaced both: the x
// gathers still cost every consumer warp an exposed L2 / DRAM round trip per tile, and 34
// warps per SM do not cover it.

// K1 for matrices whose slices are all diagonal (the stencil configs c1, c3, c4, c5): the same
// SELL-32 row sums with the matrix streamed by the bulk-copy engine.  Persistent CTAs, CPS
// per SM, of CW consumer warps + 1 producer warp; tile = CW slices (32 CW rows).  Per tile
// the producer issues four bulk copies into a shared-memory ring stage -- the tile's values
// (contiguous in the SELL copy, at most 8 per row), its row lengths, masks and slice offset
// lists -- completion counted on the stage's mbarrier, and leaves each slice's offset inside
// the stage next to them.  Consumer warp w owns slice w of every tile (thread = row): it
// picks its column offsets from the list in shared memory (no shuffles), issues the x
// gathers (L1 / L2: a stencil's neighbours), takes its values from the stage, releases the
// stage, and sums in the row's CSR order with separate multiply and add (bitwise the
// oracle's row loop).  The DRAM stream (8 B per nonzero + 2 B per row) no longer waits on a
// chain of dependent loads per warp (lengths -> values -> gathers): SP_STAGES tiles per CTA
// are always in flight.
template <int CW>
struct SellPipe {
    static constexpr int THREADS = (CW + 1) * 32;
    static constexpr int ROWS = CW * 32;
    static constexpr int VAL_BYTES = ROWS * 8 * (int)sizeof(double);  // <= 8 entries per row
    static constexpr int STAGE_BYTES = VAL_BYTES + 3 * ROWS + CW * (int)sizeof(int);  // + len, mask, diag, slice offsets
};

template <int CW, int STAGES, int CPS, bool RESID>
__global__ void __launch_bounds__(SellPipe<CW>::THREADS, CPS)
    spmv_sell_pipe_kernel(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ diag,
                          const uint8_t* __restrict__ len8, const uint8_t* __restrict__ mask8,
                          const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                          const double* __restrict__ b, const int* istate) {
    using P = SellPipe<CW>;
    if (!running(istate)) return;  // uniform: before any barrier is initialised
    extern __shared__ __align__(128) unsigned char smem_sp[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_sp + (size_t)STAGES * P::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) { mbar_init(full + s, 1); mbar_init(empty + s, CW); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t ns = (nrows + 31) / 32;
    const int64_t ntiles = (ns + CW - 1) / CW;
    const int64_t nk = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (warp == CW) {
        // ---------------- producer warp: lanes 0..CW read the slice offsets of the tile, one
        // tile ahead; lane 0 issues the copies ----------------
        auto load_ptr = [&](int64_t k) -> int64_t {
            if (k >= nk || lane > CW) return 0;
            const int64_t s = min((blockIdx.x + k * (int64_t)gridDim.x) * CW + lane, ns);
            return __ldg(ptr + s);
        };
        int64_t pn = load_ptr(0);
        for (int64_t k = 0; k < nk; k++) {
            const int64_t pc = pn;
            pn = load_ptr(k + 1);
            const int st = (int)(k % STAGES);
            unsigned char* stage = smem_sp + (size_t)st * P::STAGE_BYTES;
            const int64_t s0 = (blockIdx.x + k * (int64_t)gridDim.x) * CW;
            const int nsl = (int)min((int64_t)CW, ns - s0);
            const int64_t e0 = __shfl_sync(FULL_MASK, pc, 0), e1 = __shfl_sync(FULL_MASK, pc, nsl);
            if (lane == 0) mbar_wait(empty + st, (uint32_t)(((k / STAGES) & 1) ^ 1));
            __syncwarp();
            if (lane < CW) reinterpret_cast<int*>(stage + P::VAL_BYTES + 3 * P::ROWS)[lane] = (int)(pc - e0);
            __syncwarp();
            if (lane == 0) {
                const uint32_t vb = (uint32_t)((e1 - e0) * (int64_t)sizeof(double)), mb = (uint32_t)nsl * 32u;
                mbar_arrive_expect_tx(full + st, vb + 3u * mb);  // release: the offsets above are visible
                if (vb) bulk_g2s(stage, val + e0, vb, full + st);
                bulk_g2s(stage + P::VAL_BYTES, len8 + 32 * s0, mb, full + st);
                bulk_g2s(stage + P::VAL_BYTES + P::ROWS, mask8 + 32 * s0, mb, full + st);
                bulk_g2s(stage + P::VAL_BYTES + 2 * P::ROWS, diag + 8 * s0, mb, full + st);
            }
        }
    } else {
        // ---------------- consumer warp w: slice w of every tile ----------------
        for (int64_t k = 0; k < nk; k++) {
            const int st = (int)(k % STAGES);
            const unsigned char* stage = smem_sp + (size_t)st * P::STAGE_BYTES;
            const int64_t s0 = (blockIdx.x + k * (int64_t)gridDim.x) * CW;
            const int64_t r = (s0 + warp) * 32 + lane;
            const bool have = s0 + warp < ns;  // warp-uniform (slices past the end were not copied)
            mbar_wait(full + st, (uint32_t)((k / STAGES) & 1));
            int len = have ? (int)stage[P::VAL_BYTES + 32 * warp + lane] : 0;  // rows >= nrows: padded with 0
            const bool bnd = (len == SELL_BOUNDARY);  // G > 1 boundary row: launch_spmv_rows, after the halo
            if (bnd) len = 0;
            const unsigned m = (have && !bnd) ? (unsigned)stage[P::VAL_BYTES + P::ROWS + 32 * warp + lane] : 0u;
            const int4* dg = reinterpret_cast<const int4*>(stage + P::VAL_BYTES + 2 * P::ROWS + 32 * warp);
            const int4 d0 = dg[0], d1 = dg[1];
            const int dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
            const double* vs = reinterpret_cast<const double*>(stage) +
                               reinterpret_cast<const int*>(stage + P::VAL_BYTES + 3 * P::ROWS)[warp] + lane;
            const char* xb = reinterpret_cast<const char*>(x + r);
            double xv[8], vv[8];
            // list position j in order = the row's CSR order (see sell_row)
#pragma unroll
            for (int j = 0; j < 8; j++) xv[j] = ((m >> j) & 1u) ? __ldg(reinterpret_cast<const double*>(xb + 8 * (int64_t)dd[j])) : 0.0;
            double bv = 0.0;
            if (RESID && m) bv = __ldg(b + r);
#pragma unroll
            for (int j = 0; j < 8; j++) vv[j] = ((m >> j) & 1u) ? vs[32 * j] : 0.0;
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);  // the stage refills while the gathers are in flight
            double sum = 0.0;  // absent positions add 0.0 * 0.0 = +0.0: no bit of the sum changes (sell_row)
#pragma unroll
            for (int j = 0; j < 8; j++) sum = __dadd_rn(sum, __dmul_rn(vv[j], xv[j]));
            if (have && r < nrows && !bnd) {
                if (RESID && !m) bv = __ldg(b + r);
                y[r] = RESID ? bv - sum : sum;
            }
        }
    }
}

template <int CW, int STAGES, int CPS>
static bool spmv_sell_pipe(const SpmvArgs& a, const double* x, double* y, const double* b, bool resid,
                           const int* istate, cudaStream_t s) {
    using P = SellPipe<CW>;
    static int sms = 0;
    static bool ok = false;
    const size_t smem = (size_t)STAGES * P::STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        ok = cudaFuncSetAttribute(spmv_sell_pipe_kernel<CW, STAGES, CPS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
             cudaFuncSetAttribute(spmv_sell_pipe_kernel<CW, STAGES, CPS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
        if (!ok) cudaGetLastError();
    }
    if (!ok) return false;
    const int64_t ntiles = ((a.nrows + 31) / 32 + CW - 1) / CW;
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, CPS * (int64_t)sms);
    if (resid) spmv_sell_pipe_kernel<CW, STAGES, CPS, true><<<grid, P::THREADS, smem, s>>>(a.nrows, a.sell_ptr, a.sell_diag, a.sell_len, a.sell_mask, a.sell_val, x, y, b, istate);
    else spmv_sell_pipe_kernel<CW, STAGES, CPS, false><<<grid, P::THREADS, smem, s>>>(a.nrows, a.sell_ptr, a.sell_diag, a.sell_len, a.sell_mask, a.sell_val, x, y, b, istate);
    return true;
}

