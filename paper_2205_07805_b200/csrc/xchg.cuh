// Fused block dot + allreduce over NVLink peer memory: the last CTA of
// the block-dot kernel, having summed its rank's partials, writes the 2(p+1) local dots into
// its slot of an NCCL symmetric window, meets the other ranks at an LSA (load/store
// accessible) barrier of the NCCL 2.28 device API, and sums the G slots in rank order
// 0..G-1 with direct loads from the peers' windows.  Every rank computes the same sum in
// the same order, so the reduced vector is bitwise identical on all ranks (the small step
// is replicated from it, §8(e)), and no separate ncclAllReduce launch sits between the
// block dot and the small step.
//
// Two slots alternate by call parity: a rank can only write slot s of call c+2 after it
// passed the barrier of call c+1, which every peer reaches only after it finished reading
// the slots of call c.  All ranks issue the same sequence of block dots (SPMD), so the
// parity and the barrier epochs agree.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "ptx_util.cuh"

namespace igs {

struct XchgDev {
    ncclDevComm comm;   // device communicator (LSA team = all ranks)
    ncclWindow_t win;   // symmetric window, 2 slots of slot_doubles
    unsigned* calls;    // device call counter (slot parity)
    int slot_doubles;
    int nranks;
};

// Stage 2 of the block dot with the cross-rank sum fused in (last CTA only, all threads).
__device__ __forceinline__ void final_reduce_xchg(const double* __restrict__ part, int stride, int nparts,
                                                  double* out, const XchgDev& x) {
    const unsigned call = *(volatile unsigned*)x.calls;
    const size_t off = (size_t)(call & 1u) * (size_t)x.slot_doubles * sizeof(double);
    double* mine = static_cast<double*>(ncclGetLocalPointer(x.win, off));
    final_reduce(part, stride, nparts, mine);  // this rank's sums, in CTA order
    {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), x.comm, ncclTeamTagLsa(), 0);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);  // release mine, acquire the peers'
    }
    for (int i = threadIdx.x; i < stride; i += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < x.nranks; r++)
            s += __ldcv(static_cast<const double*>(ncclGetLsaPointer(x.win, off, r)) + i);
        out[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *x.calls = call + 1u;
}

}  // namespace igs
