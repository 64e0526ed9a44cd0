// Fused block dot + allreduce over NVLink peer memory (the single
// "Global Synchronization" of Alg. 3 Step 4): the finisher CTAs of a
// reduction kernel, having summed their rank's per-CTA partials, write the local sums into
// this rank's slot of an NCCL symmetric window; the last finisher meets the other ranks at
// a barrier over the same window and sums the G slots in LSA-rank order 0..G-1 with direct
// NVLink loads.  Every rank computes the same sum in the same order, so the reduced vector
// is bitwise identical on all ranks (the small step is replicated from it),
// and no separate ncclAllReduce launch sits between the block dot and the small step.
//
// Window layout: [slot 0 | slot 1 | inbox[G] (uint32)].  Slots alternate by call parity: a
// rank can only write slot s of call c+2 after it passed the barrier of call c+1, which
// every peer reaches only after it finished reading the slots of call c.  All ranks issue
// the same sequence of exchanges (SPMD: reduction kernels never skip the exchange, even when
// the device status word says the cycle has stopped), so the parity and the epochs agree.
//
// Barrier: rank r stores epoch = call + 1 into inbox[r] of every peer (st.release.sys over
// NVLink) and spins on its own inbox[q] (ld.acquire.sys) until every peer's epoch arrived.
// The spin is bounded by timeout_ns (%globaltimer): a peer that never arrives sets *err,
// the reduced vector becomes NaN (the small step then stops the cycle) and later exchanges
// skip the barrier; the host reports IGS_ERR_NCCL instead of hanging.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "ptx_util.cuh"

namespace igs {

struct XchgDev {
    ncclDevComm comm;       // device communicator (LSA team = all ranks)
    ncclWindow_t win;       // symmetric window: 2 slots of slot_doubles + inbox[nranks]
    unsigned* calls;        // device call counter (slot parity, barrier epoch)
    int* err;               // device error word: 1 = barrier timeout
    unsigned long long timeout_ns;
    unsigned stall_call;    // test hook: the barrier of this call waits for an epoch nobody sends
    int slot_doubles;
    int nranks;             // LSA team size (== communicator size)
    int me;                 // this rank's LSA index
    size_t inbox_off;       // byte offset of inbox[0] in the window
};

__device__ __forceinline__ unsigned long long xchg_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double* xchg_slot(const XchgDev& x, unsigned call) {
    const size_t off = (size_t)(call & 1u) * (size_t)x.slot_doubles * sizeof(double);
    return static_cast<double*>(ncclGetLocalPointer(x.win, off));
}

// Cross-rank part (one CTA, all threads; this rank's sums already in xchg_slot(x, call) and
// visible at system scope): barrier, then out[i] = sum over ranks in LSA order.
__device__ __forceinline__ void xchg_finish(int stride, double* out, const XchgDev& x, unsigned call) {
    __shared__ int s_fail;
    const size_t off = (size_t)(call & 1u) * (size_t)x.slot_doubles * sizeof(double);
    if (threadIdx.x == 0) s_fail = *(volatile int*)x.err;
    __syncthreads();
    if (!s_fail) {
        const unsigned epoch = call + 1u;
        const int q = threadIdx.x;
        if (q < x.nranks && q != x.me) {  // arrive: my epoch into every peer's inbox[me]
            unsigned* dst = static_cast<unsigned*>(ncclGetLsaPointer(x.win, x.inbox_off + sizeof(unsigned) * x.me, q));
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
        }
        if (q < x.nranks && (q != x.me || call == x.stall_call)) {  // wait: every peer's epoch in my inbox
            const unsigned want = (call == x.stall_call) ? epoch + 0x40000000u : epoch;
            const unsigned* src = static_cast<const unsigned*>(ncclGetLocalPointer(x.win, x.inbox_off + sizeof(unsigned) * q));
            const unsigned long long t0 = xchg_now();
            for (;;) {
                unsigned v;
                asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(src) : "memory");
                if ((int)(v - want) >= 0) break;
                if (xchg_now() - t0 > x.timeout_ns) { atomicExch(x.err, 1); s_fail = 1; break; }
            }
        }
        __syncthreads();
    }
    const bool fail = s_fail != 0;
    for (int i = threadIdx.x; i < stride; i += blockDim.x) {
        double s = 0.0;
        if (fail) s = __longlong_as_double(0x7ff8000000000000LL);  // NaN: the small step stops
        else
            for (int r = 0; r < x.nranks; r++)
                s += __ldcv(static_cast<const double*>(ncclGetLsaPointer(x.win, off, r)) + i);
        out[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *x.calls = call + 1u;
}

// Single-finisher form (stage 2 done by one CTA): this rank's sums in CTA order into its
// slot, then the cross-rank part.
__device__ __forceinline__ void final_reduce_xchg(const double* __restrict__ part, int stride, int nparts,
                                                  double* out, const XchgDev& x) {
    const unsigned call = *(volatile unsigned*)x.calls;
    final_reduce(part, stride, nparts, xchg_slot(x, call));
    __threadfence_system();
    __syncthreads();
    xchg_finish(stride, out, x, call);
}

}  // namespace igs
