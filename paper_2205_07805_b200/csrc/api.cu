// api.cu -- host side of libigs: the C ABI of include/igs.h, the restarted IGS-GMRES
// driver, NCCL plumbing (one allreduce per iteration + halo send/recv) and per-kernel
// timing.  Device work lives in kernels.cu.
//
// P:n = PAPER.md line n (arXiv 2205.07805).  Driver semantics: SURVEY §8(c) "Driver";
// per-iteration structure: Alg. 3 for gs_iters = 2, Alg. 2 without Steps
// 14-16 for gs_iters = 1.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <map>
#include <utility>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/igs.h"
#include "igs_internal.cuh"
#include "sell_plan.h"
#include "xchg.cuh"

namespace igs {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace igs

using namespace igs;

#define CUDA_TRY(x)                                                                        \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            set_error(std::string(#x) + " failed: " + cudaGetErrorString(e_));            \
            return e_ == cudaErrorMemoryAllocation ? IGS_ERR_OOM : IGS_ERR_CUDA;           \
        }                                                                                  \
    } while (0)
#define NCCL_TRY(x)                                                                        \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess) {                                                           \
            set_error(std::string(#x) + " failed: " + ncclGetErrorString(r_));            \
            return IGS_ERR_NCCL;                                                           \
        }                                                                                  \
    } while (0)
#define TRY(x)                        \
    do {                              \
        igs_status s_ = (x);          \
        if (s_ != IGS_OK) return s_;  \
    } while (0)
#define ARG_CHECK(cond, msg)              \
    do {                                  \
        if (!(cond)) {                    \
            set_error(std::string(msg));  \
            return IGS_ERR_ARG;           \
        }                                 \
    } while (0)

struct TimedLaunch {
    int kind;
    double bytes;
    int ev0, ev1;
};

struct igs_ctx {
    int dev = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // small-step tail (H, Givens, status), overlapped with the update
    cudaStream_t gstream = nullptr;  // private stream for CUDA-graph capture/replay
    cudaEvent_t ev_g0 = nullptr, ev_g1 = nullptr;
    cudaEvent_t ev_crit = nullptr, ev_tail = nullptr;
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;
    int num_sms = 148;
    bool ok = false;

    int64_t n_global = 0, row_begin = 0, n_local = 0, ldv = 0;
    // matrix, local column space [0, n_local + n_ghost)
    SpmvArgs A{};
    void* d_rowptr = nullptr;
    void* d_col = nullptr;
    double* d_val = nullptr;
    int64_t nnz = 0;
    bool csr_compact = false;  // CSR arrays hold only the boundary rows (a SELL copy exists)
    // halo
    int64_t n_ghost = 0;
    double* d_ghost = nullptr;
    double* d_send = nullptr;
    int64_t* d_send_idx = nullptr;
    int64_t n_send = 0;
    std::vector<int> peers;
    std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
    // workspace
    int m_cap = 0, k_cap = 0;
    double* d_V = nullptr;
    double* d_z = nullptr;
    double* d_b = nullptr;
    double* d_x = nullptr;
    double* d_small = nullptr;  // all small double arrays
    int* d_int = nullptr;
    double* d_part = nullptr;
    unsigned* d_counter = nullptr;
    double* d_gram = nullptr;  // gram partials + G
    size_t gram_cap = 0;
    int bdot_grid = 1;
    int part_rows = 1;  // capacity of d_part in rows (>= every reduction grid)
    Dev dev_state{};
    double* h_pinned = nullptr;  // small pinned staging
    int* h_pinned_int = nullptr;
    void* bound_ws = nullptr;
    size_t bound_bytes = 0;
    bool owns_ws = true;
    // counters
    int64_t n_allreduce = 0, n_halo = 0, n_iter = 0, n_reduce = 0;
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> events;
    std::vector<TimedLaunch> recs;
    double t_ms[IGS_K_COUNT] = {0};
    double t_bytes[IGS_K_COUNT] = {0};
    int64_t t_launch[IGS_K_COUNT] = {0};
    int64_t tail_launches = 0;  // side-stream small-step tails (untimed)
    // CUDA graphs of whole restart cycles (small problems, single GPU, timing off)
    bool graphs_enabled = true;
    bool capturing = false;
    struct CycleGraph {
        cudaGraphExec_t exec;
        int64_t reductions, allreduces, halos;  // counters one replay accounts for
    };
    std::map<std::pair<int, int>, CycleGraph> graphs;  // (m, alg) -> executable cycle
    int64_t n_graph_launches = 0;
    // persistent cycle kernel (small n, single GPU, Alg. 3 / Alg. 2 one sweep)
    bool pc_enabled = true;   // IGS_PERSIST=0 disables
    bool mgs_fused = true;    // IGS_MGS_FUSED=0: MGS with separate dot and axpy kernels
    bool xs_enabled = true;   // IGS_PC_XSTAGE=0: persistent kernel gathers u from L2 (long rows)
    int last_ares = 0;        // resident-A entries per CTA of the last persistent launch (0: not resident)
    bool ares_enabled = true; // IGS_PC_ARES=0: persistent kernel re-reads A from L2 every iteration
    std::vector<int32_t> h_rowlen;  // row lengths (n <= pcycle_xs_max(), no SELL copy): sizes the resident A
    bool two_fused = true;    // IGS_TWO_FUSED=0: Alg. 2 two-reduce with a separate second block dot
    double two_fused_l2 = 80e6;  // IGS_TWO_FUSED_L2_MB: L2 budget of the fused update + dot
    int pc_ntri = 0;          // IGS_PC_NTRI: forward-substitution CTAs of the persistent kernel (0 = auto)
    // crossover with the graph-replayed per-kernel path, per algorithm (m = 100 and 300,
    // profiles/r2/pc_crossover.jsonl): Alg. 3 ahead through n = 196249 (1.02 / 1.16), behind
    // from 262144; IGS(1) ahead through 90000 (1.16 / 1.28), behind from 147456.
    // IGS_PC_MAX_N overrides both.
    int64_t pc_max_n = -1;
    int pc_grid = 0;          // IGS_PC_GRID overrides the size heuristic
    int64_t pc_rowsplit_n = 4096;  // IGS_PC_ROWSPLIT_N: row-block dots from this many rows
    int64_t n_pcycle = 0;
    unsigned long long* d_pcprof = nullptr;  // IGS_PC_PROF=1 phase timestamps

    // SELL-32 copy of A (short rows)
    int64_t* d_sell_ptr = nullptr;
    uint8_t* d_sell_len = nullptr;
    double* d_sell_val = nullptr;
    void* d_sell_col = nullptr;
    int64_t* d_sell_cptr = nullptr;
    int32_t* d_sell_diag = nullptr;
    uint8_t* d_sell_mask = nullptr;
    int64_t sell_entries = 0, sell_diag_slices = 0, sell_stream_bytes = 0;
    // G > 1 with SELL: rows touching ghost columns run after the halo, the rest during it
    int64_t* d_bnd_rows = nullptr;
    cudaStream_t hstream = nullptr;  // halo exchange stream
    cudaStream_t cstream = nullptr;  // host-vector solves: D2H of x chunks behind the last x update
    cudaEvent_t ev_xc[8] = {};
    cudaEvent_t ev_x = nullptr, ev_h = nullptr;
    // fused block dot + allreduce over NVLink (IGS_XCHG=1): NCCL symmetric window + device comm
    bool xchg_req = false;
    bool force_nccl = false;  // IGS_FORCE_NCCL=1: a 1-rank communicator and real ncclAllReduce calls
    void* xbuf = nullptr;
    ncclWindow_t xwin = nullptr;
    ncclDevComm dcomm{};
    bool dcomm_ok = false;
    XchgDev* d_xchg = nullptr;  // device copy; null = separate ncclAllReduce
    XchgDev h_xchg{};           // host copy (timeout / test-hook updates are re-uploaded)
    int* d_misc = nullptr;      // [0]: agreement flag (agree_all), [1]: exchange error word
    int* d_xerr = nullptr;      // = d_misc + 1: 1 after an exchange barrier timeout
    int xslot = 0;              // slot capacity (doubles) of the registered window
    // failure handling: host waits poll ncclCommGetAsyncError and give up after
    // timeout_s (ncclCommAbort); the exchange barrier has the same device-side bound
    double timeout_s = 120.0;   // IGS_NCCL_TIMEOUT_S / igs_set_timeout
    bool aborted = false;       // communicator aborted: the context only accepts igs_destroy
    // virtual ranks (igs_create_virtual, test hook): G contexts of one process on one device;
    // the halo copies from the owning context's send buffer instead of NCCL send/recv
    struct VGroup* vgroup = nullptr;
    // igs_virtual_solve: the member runs igs_solve on its own host thread and stream; its
    // collectives are emulated (vallreduce / vhalo: host barrier + cross-stream events +
    // device copies, no device-side waiting between members)
    bool vsolve = false;
    uint64_t v_ar_calls = 0, v_halo_calls = 0;
    double* d_vstage = nullptr;  // [2][vstage_cap] allreduce staging (call parity)
    size_t vstage_cap = 0;
};

// ------------------------------------------------------------------------------ misc
extern "C" const char* igs_last_error(void) { return g_err.c_str(); }

static inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

static igs_status timer_begin(igs_ctx* c, int* idx, cudaStream_t st) {
    *idx = -1;
    if (!c->timing || c->capturing) return IGS_OK;
    const size_t need = 2 * (c->recs.size() + 1);
    while (c->events.size() < need) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreate(&e));
        c->events.push_back(e);
    }
    *idx = (int)(2 * c->recs.size());
    CUDA_TRY(cudaEventRecord(c->events[*idx], st));
    c->recs.push_back({-1, 0.0, *idx, *idx + 1});  // reserve the pair
    return IGS_OK;
}

static igs_status timer_end(igs_ctx* c, int idx, int kind, double bytes, cudaStream_t st) {
    if (idx < 0) return IGS_OK;
    CUDA_TRY(cudaEventRecord(c->events[idx + 1], st));
    c->recs[idx / 2] = {kind, bytes, idx, idx + 1};
    return IGS_OK;
}

static igs_status timer_flush(igs_ctx* c) {
    for (const auto& r : c->recs) {
        if (r.kind < 0) continue;
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->events[r.ev0], c->events[r.ev1]));
        c->t_ms[r.kind] += ms;
        c->t_bytes[r.kind] += r.bytes;
        c->t_launch[r.kind] += 1;
    }
    c->recs.clear();
    return IGS_OK;
}

#define TIMED_ON(strm, kind, bytes, launch_stmt)         \
    do {                                                  \
        int ti_;                                          \
        TRY(timer_begin(ctx, &ti_, (strm)));              \
        launch_stmt;                                      \
        CUDA_TRY(cudaGetLastError());                     \
        TRY(timer_end(ctx, ti_, (kind), (bytes), (strm)));\
    } while (0)
#define TIMED(kind, bytes, launch_stmt) TIMED_ON(ctx->stream, kind, bytes, launch_stmt)

// ------------------------------------------------------------- waits with a deadline
// Failure detection: with a communicator every host wait polls instead of
// blocking.  An asynchronous NCCL error (ncclCommGetAsyncError) or no progress for
// ctx->timeout_s (a peer rank died or never joined a collective) aborts the communicator
// (ncclCommAbort) and returns IGS_ERR_NCCL; the context then only accepts igs_destroy.
// The fused exchange's barrier is bounded on the device by the same timeout (xchg.cuh).
static igs_status abort_comm(igs_ctx* ctx, const std::string& why) {
    if (ctx->comm && !ctx->aborted) ncclCommAbort(ctx->comm);
    ctx->aborted = true;
    ctx->ok = false;
    set_error(why + " (communicator aborted; destroy the context)");
    return IGS_ERR_NCCL;
}

static igs_status wait_for(igs_ctx* ctx, cudaEvent_t ev, cudaStream_t st, const char* what) {
    if (!ctx->comm) {
        const cudaError_t e = ev ? cudaEventSynchronize(ev) : cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            set_error(std::string(what) + ": " + cudaGetErrorString(e));
            return IGS_ERR_CUDA;
        }
        return IGS_OK;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; spin++) {
        const cudaError_t q = ev ? cudaEventQuery(ev) : cudaStreamQuery(st);
        if (q == cudaSuccess) return IGS_OK;
        if (q != cudaErrorNotReady) {
            set_error(std::string(what) + ": " + cudaGetErrorString(q));
            return IGS_ERR_CUDA;
        }
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(ctx->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
            return abort_comm(ctx, std::string(what) + ": NCCL asynchronous error: " + ncclGetErrorString(ar));
        if ((spin & 255u) == 255u) {
            const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            // twice the device bound of the exchange barrier (xchg.cuh, timeout_s): a peer that
            // stops arriving there is reported by the device path ("barrier timeout"); the
            // host deadline catches what the device cannot see (send/recv, NCCL kernels)
            if (el > 2.0 * ctx->timeout_s)
                return abort_comm(ctx, std::string(what) + ": timeout, no progress for " +
                                           std::to_string(ctx->timeout_s) + " s (a peer rank stopped or hung?)");
        }
        if (spin >= 1024) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

// --------------------------------------------------------------------- create / destroy
extern "C" igs_status igs_nccl_unique_id(void* out128) {
    ARG_CHECK(out128 != nullptr, "igs_nccl_unique_id: NULL output");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return IGS_OK;
}

static igs_status validate_csr(int64_t n_global, int64_t n_local, const int64_t* rowptr,
                               const void* colind, int bits, const double* values, int64_t nnz) {
    ARG_CHECK(rowptr[0] == 0, "igs_create: rowptr[0] != 0");
    ARG_CHECK(rowptr[n_local] == nnz, "igs_create: rowptr[n_local] != nnz_local");
    for (int64_t i = 0; i < n_local; i++) {
        ARG_CHECK(rowptr[i + 1] >= rowptr[i], "igs_create: rowptr not monotone");
        int64_t prev = -1;
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; q++) {
            const int64_t cc = bits == 64 ? static_cast<const int64_t*>(colind)[q]
                                          : (int64_t) static_cast<const int32_t*>(colind)[q];
            ARG_CHECK(cc >= 0 && cc < n_global, "igs_create: column index out of range");
            ARG_CHECK(cc > prev, "igs_create: column indices not strictly increasing in a row");
            prev = cc;
        }
    }
    for (int64_t q = 0; q < nnz; q++)
        if (!std::isfinite(values[q])) {
            set_error("igs_create: non-finite matrix entry");
            return IGS_ERR_NONFINITE;
        }
    return IGS_OK;
}

// Virtual ranks (igs_create_virtual): the row bounds and every rank's ghost list are known
// on the host, so the two all-gathers and the request exchange of setup_halo are computed.
struct VirtPlan {
    std::vector<int64_t> bounds;               // [G + 1]
    std::vector<std::vector<int64_t>> ghosts;  // ghosts[q]: rank q's ghost columns (ascending)
};
struct VGroup {
    int G = 0;
    std::vector<igs_ctx*> members;
    int alive = 0;
    // igs_virtual_solve: a host barrier per emulated collective (members enqueue, then meet),
    // and per (call parity, member) events: staged copy done, sum done, pack done, ghost
    // copies done
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    double timeout_s = 120.0;
    std::vector<cudaEvent_t> ev_copy[2], ev_sum[2], ev_pack, ev_hcopy;
    const double** d_stage_ptrs = nullptr;  // [2][G] device array of the members' staging slots
    ~VGroup() {
        for (int q = 0; q < 2; q++) {
            for (cudaEvent_t e : ev_copy[q]) cudaEventDestroy(e);
            for (cudaEvent_t e : ev_sum[q]) cudaEventDestroy(e);
        }
        for (cudaEvent_t e : ev_pack) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_hcopy) cudaEventDestroy(e);
        if (d_stage_ptrs) cudaFree(d_stage_ptrs);
    }
    // all G members arrive (enqueue-time rendezvous); false if a member failed or time ran out
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const uint64_t g0 = gen;
        if (++arrived == G) {
            arrived = 0;
            gen++;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g0 || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
    void fail() {
        std::lock_guard<std::mutex> lk(mu);
        broken = true;
        cv.notify_all();
    }
};

static igs_status setup_halo(igs_ctx* ctx, const int64_t* rowptr, const void* colind, int bits,
                             std::vector<int64_t>& local_col, const VirtPlan* vp) {
    const int G = ctx->nranks;
    std::vector<int64_t> bounds(G + 1, 0);
    if (vp) {
        bounds = vp->bounds;
    } else if (G > 1) {
        // all-gather (row_begin, n_local) through NCCL
        int64_t* d_bl = nullptr;
        CUDA_TRY(cudaMalloc(&d_bl, sizeof(int64_t) * 2 * G));
        int64_t mine[2] = {ctx->row_begin, ctx->n_local};
        CUDA_TRY(cudaMemcpyAsync(d_bl + 2 * ctx->rank, mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
        NCCL_TRY(ncclAllGather(d_bl + 2 * ctx->rank, d_bl, 2, ncclInt64, ctx->comm, ctx->stream));
        std::vector<int64_t> bl(2 * G);
        CUDA_TRY(cudaMemcpyAsync(bl.data(), d_bl, sizeof(int64_t) * 2 * G, cudaMemcpyDeviceToHost, ctx->stream));
        TRY(wait_for(ctx, nullptr, ctx->stream, "igs_create: halo plan"));
        cudaFree(d_bl);
        for (int q = 0; q < G; q++) {
            ARG_CHECK(bl[2 * q] == (q == 0 ? 0 : bl[2 * (q - 1)] + bl[2 * (q - 1) + 1]),
                      "igs_create: row blocks do not tile [0, n) in rank order");
            bounds[q] = bl[2 * q];
        }
        bounds[G] = bl[2 * (G - 1)] + bl[2 * (G - 1) + 1];
        ARG_CHECK(bounds[G] == ctx->n_global, "igs_create: row blocks do not cover n_global");
    } else {
        ARG_CHECK(ctx->row_begin == 0 && ctx->n_local == ctx->n_global,
                  "igs_create: single rank must own all rows");
        bounds[1] = ctx->n_global;
    }
    int64_t ng = 0;
    std::vector<int64_t> owner_cnt(G, 0);
    TRY(igs_plan_ghosts(ctx->row_begin, ctx->n_local, rowptr, colind, bits, G, bounds.data(), &ng,
                        nullptr, owner_cnt.data()));
    std::vector<int64_t> ghosts(ng);
    TRY(igs_plan_ghosts(ctx->row_begin, ctx->n_local, rowptr, colind, bits, G, bounds.data(), &ng,
                        ghosts.data(), owner_cnt.data()));
    local_col.resize(ctx->n_local > 0 ? rowptr[ctx->n_local] : 0);
    TRY(igs_plan_remap(ctx->row_begin, ctx->n_local, rowptr, colind, bits, ng, ghosts.data(),
                       local_col.data()));
    ctx->n_ghost = ng;
    if (G == 1) {
        ARG_CHECK(ng == 0, "igs_create: ghost columns with one rank");
        return IGS_OK;
    }
    // count matrix cnt[q][r] = ghosts rank q needs from rank r (all-gather of owner counts)
    std::vector<int64_t> cnt((size_t)G * G, 0);
    if (vp) {
        for (int q = 0; q < G; q++)
            for (int64_t c : vp->ghosts[q]) {
                const int r = (int)(std::upper_bound(bounds.begin(), bounds.end(), c) - bounds.begin()) - 1;
                cnt[(size_t)q * G + r]++;
            }
    } else {
        int64_t* d_cnt = nullptr;
        CUDA_TRY(cudaMalloc(&d_cnt, sizeof(int64_t) * G * G));
        CUDA_TRY(cudaMemcpyAsync(d_cnt + (int64_t)G * ctx->rank, owner_cnt.data(), sizeof(int64_t) * G,
                                 cudaMemcpyHostToDevice, ctx->stream));
        NCCL_TRY(ncclAllGather(d_cnt + (int64_t)G * ctx->rank, d_cnt, G, ncclInt64, ctx->comm, ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int64_t) * G * G, cudaMemcpyDeviceToHost, ctx->stream));
        TRY(wait_for(ctx, nullptr, ctx->stream, "igs_create: halo plan"));
        cudaFree(d_cnt);
    }
    // receive side: my ghosts, grouped by owner (ghosts are sorted, owners ascending)
    // send side: rows other ranks need from me
    ctx->peers.clear(); ctx->send_off.clear(); ctx->send_cnt.clear(); ctx->recv_off.clear(); ctx->recv_cnt.clear();
    int64_t roff = 0, soff = 0;
    for (int q = 0; q < G; q++) {
        const int64_t rc = cnt[(size_t)ctx->rank * G + q];  // I need rc from q
        const int64_t sc = cnt[(size_t)q * G + ctx->rank];  // q needs sc from me
        if (q == ctx->rank) { ARG_CHECK(rc == 0, "igs_create: self ghost"); continue; }
        if (rc == 0 && sc == 0) continue;
        ctx->peers.push_back(q);
        ctx->recv_off.push_back(roff); ctx->recv_cnt.push_back(rc); roff += rc;
        ctx->send_off.push_back(soff); ctx->send_cnt.push_back(sc); soff += sc;
    }
    ctx->n_send = soff;
    // exchange the requested global indices
    std::vector<int64_t> req(soff);
    if (vp) {  // the peers' requests, in peer order: peer q's ghosts that I own
        int64_t at = 0;
        for (size_t i = 0; i < ctx->peers.size(); i++)
            for (int64_t c : vp->ghosts[ctx->peers[i]])
                if (c >= ctx->row_begin && c < ctx->row_begin + ctx->n_local) req[(size_t)at++] = c;
        ARG_CHECK(at == soff, "igs_create_virtual: inconsistent halo plan");
    } else {
    int64_t *d_req_out = nullptr, *d_req_in = nullptr;
    CUDA_TRY(cudaMalloc(&d_req_out, sizeof(int64_t) * std::max<int64_t>(ng, 1)));
    CUDA_TRY(cudaMalloc(&d_req_in, sizeof(int64_t) * std::max<int64_t>(soff, 1)));
    CUDA_TRY(cudaMemcpyAsync(d_req_out, ghosts.data(), sizeof(int64_t) * ng, cudaMemcpyHostToDevice, ctx->stream));
    NCCL_TRY(ncclGroupStart());
    for (size_t i = 0; i < ctx->peers.size(); i++) {
        if (ctx->recv_cnt[i]) NCCL_TRY(ncclSend(d_req_out + ctx->recv_off[i], ctx->recv_cnt[i], ncclInt64, ctx->peers[i], ctx->comm, ctx->stream));
        if (ctx->send_cnt[i]) NCCL_TRY(ncclRecv(d_req_in + ctx->send_off[i], ctx->send_cnt[i], ncclInt64, ctx->peers[i], ctx->comm, ctx->stream));
    }
    NCCL_TRY(ncclGroupEnd());
    CUDA_TRY(cudaMemcpyAsync(req.data(), d_req_in, sizeof(int64_t) * soff, cudaMemcpyDeviceToHost, ctx->stream));
    TRY(wait_for(ctx, nullptr, ctx->stream, "igs_create: halo plan"));
    cudaFree(d_req_out);
    cudaFree(d_req_in);
    }
    for (auto& r : req) {
        ARG_CHECK(r >= ctx->row_begin && r < ctx->row_begin + ctx->n_local, "igs_create: bad halo request");
        r -= ctx->row_begin;
    }
    CUDA_TRY(cudaMalloc(&ctx->d_send_idx, sizeof(int64_t) * std::max<int64_t>(soff, 1)));
    CUDA_TRY(cudaMalloc(&ctx->d_send, sizeof(double) * std::max<int64_t>(soff, 1)));
    CUDA_TRY(cudaMalloc(&ctx->d_ghost, sizeof(double) * std::max<int64_t>(ng, 1)));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_send_idx, req.data(), sizeof(int64_t) * soff, cudaMemcpyHostToDevice, ctx->stream));
    TRY(wait_for(ctx, nullptr, ctx->stream, "igs_create: halo plan"));
    return IGS_OK;
}

static void release_xchg(igs_ctx* ctx);

static void free_ctx(igs_ctx* c) {
    if (!c) return;
    cudaFree(c->d_rowptr); cudaFree(c->d_col); cudaFree(c->d_val);
    cudaFree(c->d_ghost); cudaFree(c->d_send); cudaFree(c->d_send_idx);
    if (c->owns_ws) { cudaFree(c->d_V); }
    cudaFree(c->d_z); cudaFree(c->d_b); cudaFree(c->d_x);
    cudaFree(c->d_small); cudaFree(c->d_int); cudaFree(c->d_part); cudaFree(c->d_counter); cudaFree(c->d_pcprof);
    cudaFree(c->d_sell_ptr); cudaFree(c->d_sell_len); cudaFree(c->d_sell_val); cudaFree(c->d_sell_col);
    cudaFree(c->d_sell_cptr); cudaFree(c->d_sell_diag); cudaFree(c->d_sell_mask); cudaFree(c->d_vstage);
    cudaFree(c->d_bnd_rows);
    if (c->hstream) cudaStreamDestroy(c->hstream);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    for (cudaEvent_t e : c->ev_xc) if (e) cudaEventDestroy(e);
    if (c->ev_x) cudaEventDestroy(c->ev_x);
    if (c->ev_h) cudaEventDestroy(c->ev_h);
    cudaFree(c->d_gram);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->h_pinned_int) cudaFreeHost(c->h_pinned_int);
    for (auto e : c->events) cudaEventDestroy(e);
    if (c->ev_crit) cudaEventDestroy(c->ev_crit);
    if (c->ev_tail) cudaEventDestroy(c->ev_tail);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->gstream) cudaStreamDestroy(c->gstream);
    if (c->ev_g0) cudaEventDestroy(c->ev_g0);
    if (c->ev_g1) cudaEventDestroy(c->ev_g1);
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
    // after ncclCommAbort the communicator's resources are gone with it
    if (c->dcomm_ok && !c->aborted) ncclDevCommDestroy(c->comm, &c->dcomm);
    release_xchg(c);
    cudaFree(c->d_misc);
    if (c->comm && !c->aborted) ncclCommDestroy(c->comm);
    delete c;
}

// SELL-32 (slices of 32 rows, entries of a slice interleaved by row) from the host CSR.
static igs_status build_sell(igs_ctx* ctx, const int64_t* rowptr, const std::vector<int64_t>& local_col,
                             const double* values, bool idx64, std::vector<int64_t>& bnd) {
    const int64_t n = ctx->n_local, ns = (n + 31) / 32;
    // G > 1: rows that touch a ghost column are left to the boundary pass (row-list kernel,
    // after the halo); the SELL pass runs while the halo is in flight and skips them
    // (row length SELL_BOUNDARY, no entries stored)
    bnd.clear();
    for (int64_t r = 0; r < n && ctx->n_ghost > 0; r++)
        for (int64_t q = rowptr[r]; q < rowptr[r + 1]; q++)
            if (local_col[(size_t)q] >= n) { bnd.push_back(r); break; }
    // test hook (one GPU): IGS_TEST_BND_EVERY=k routes every k-th row through the boundary
    // pass, so the split interior / boundary SpMV of G > 1 is checked on a single device
    if (const char* e = std::getenv("IGS_TEST_BND_EVERY"))
        if (ctx->nranks == 1 && std::atoi(e) > 0)
            for (int64_t r = 0; r < n; r += std::atoi(e)) bnd.push_back(r);
    // IGS_TEST_BND_ENDS=m: the first and the last m rows instead (the shape of a z-slab's
    // boundary: its two outer planes; tools/slab_proxy.py)
    if (const char* e = std::getenv("IGS_TEST_BND_ENDS"))
        if (ctx->nranks == 1 && bnd.empty() && std::atoll(e) > 0) {
            const int64_t m = std::min<int64_t>(std::atoll(e), n / 2);
            for (int64_t r = 0; r < m; r++) bnd.push_back(r);
            for (int64_t r = n - m; r < n; r++) bnd.push_back(r);
        }
    // the slice layout is host-only work (plan.cpp, also behind igs_plan_sell for the CPU
    // tests).  Test hook IGS_SELL_DIAG=0 keeps every slice explicit.
    const char* edg = std::getenv("IGS_SELL_DIAG");
    SellHost h;
    sell_plan(n, rowptr, local_col.data(), values, bnd, !(edg && std::atoi(edg) == 0), h);
    if (!h.built) { bnd.clear(); return IGS_OK; }  // long rows: keep the CSR kernels
    const std::vector<int64_t>&sp = h.ptr, &cp = h.cptr;
    const std::vector<int32_t>& dg = h.diag;
    const std::vector<uint8_t>&len = h.len, &mk = h.mask;
    const std::vector<double>& sv = h.val;
    const int64_t tot = (int64_t)sv.size(), ctot = cp[(size_t)ns], ndiag = h.ndiag;
    std::vector<char> sc((size_t)std::max<int64_t>(ctot, 1) * (idx64 ? 8 : 4), 0);
    for (int64_t q = 0; q < ctot; q++) {
        if (idx64) reinterpret_cast<int64_t*>(sc.data())[q] = h.col[(size_t)q];
        else reinterpret_cast<int32_t*>(sc.data())[q] = (int32_t)h.col[(size_t)q];
    }
    CUDA_TRY(cudaMalloc(&ctx->d_sell_ptr, sizeof(int64_t) * sp.size()));
    CUDA_TRY(cudaMalloc(&ctx->d_sell_len, len.size()));
    CUDA_TRY(cudaMalloc(&ctx->d_sell_val, sizeof(double) * sv.size()));
    CUDA_TRY(cudaMalloc(&ctx->d_sell_col, sc.size()));
    CUDA_TRY(cudaMalloc(&ctx->d_sell_cptr, sizeof(int64_t) * cp.size()));
    CUDA_TRY(cudaMalloc(&ctx->d_sell_diag, sizeof(int32_t) * dg.size()));
    CUDA_TRY(cudaMalloc(&ctx->d_sell_mask, mk.size()));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_ptr, sp.data(), sizeof(int64_t) * sp.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_len, len.data(), len.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_val, sv.data(), sizeof(double) * sv.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_col, sc.data(), sc.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_cptr, cp.data(), sizeof(int64_t) * cp.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_diag, dg.data(), sizeof(int32_t) * dg.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(ctx->d_sell_mask, mk.data(), mk.size(), cudaMemcpyHostToDevice));
    ctx->A.sell_ptr = ctx->d_sell_ptr;
    ctx->A.sell_len = ctx->d_sell_len;
    ctx->A.sell_val = ctx->d_sell_val;
    ctx->A.sell_col = ctx->d_sell_col;
    ctx->A.sell_cptr = ctx->d_sell_cptr;
    ctx->A.sell_diag = ctx->d_sell_diag;
    ctx->A.sell_mask = ctx->d_sell_mask;
    ctx->sell_diag_slices = ndiag;
    ctx->A.sell_kind = ndiag == ns ? 1 : (ndiag == 0 ? 2 : 0);
    // test / A-B hook: row count from which an all-diagonal matrix takes the
    // slice-walking SpMV (0: always, so the tests reach it at small n; -1: never)
    if (const char* e = std::getenv("IGS_SELL_WALK_MIN_N")) ctx->A.sell_walk_min_n = std::atoll(e);
    ctx->sell_entries = tot;
    // bytes one SpMV launch streams from the SELL copy (IGS_INFO_SPMV_BYTES): stored values,
    // column indices of the explicit slices, row lengths, masks / offset lists when any slice
    // is diagonal, slice offsets; + x and y
    ctx->sell_stream_bytes = 8 * tot + (idx64 ? 8 : 4) * ctot + 32 * ns + (ndiag ? 64 * ns : 0) +
                             8 * (ns + 1) * (ndiag == ns ? 1 : 2) + 16 * n;
    if (!bnd.empty()) {
        CUDA_TRY(cudaMalloc(&ctx->d_bnd_rows, sizeof(int64_t) * bnd.size()));
        CUDA_TRY(cudaMemcpy(ctx->d_bnd_rows, bnd.data(), sizeof(int64_t) * bnd.size(), cudaMemcpyHostToDevice));
        ctx->A.bnd_rows = ctx->d_bnd_rows;
        ctx->A.n_bnd = (int64_t)bnd.size();
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->hstream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_x, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_h, cudaEventDisableTiming));
    }
    return IGS_OK;
}

static igs_status create_ctx(igs_ctx** out, int64_t n_global, int64_t row_begin,
                             int64_t n_local, const int64_t* rowptr, const void* colind,
                             int colind_bits, const double* values, int64_t nnz_local,
                             igs_mem where, int cuda_device, const void* nccl_unique_id,
                             int rank, int nranks, void* cuda_stream, const VirtPlan* vp);

extern "C" igs_status igs_create(igs_ctx** out, int64_t n_global, int64_t row_begin,
                                 int64_t n_local, const int64_t* rowptr, const void* colind,
                                 int colind_bits, const double* values, int64_t nnz_local,
                                 igs_mem where, int cuda_device, const void* nccl_unique_id,
                                 int rank, int nranks, void* cuda_stream) {
    ARG_CHECK(out != nullptr, "igs_create: NULL out");
    *out = nullptr;
    ARG_CHECK((nranks == 1) == (nccl_unique_id == nullptr), "igs_create: nccl_unique_id must be given iff nranks > 1");
    return create_ctx(out, n_global, row_begin, n_local, rowptr, colind, colind_bits, values, nnz_local, where,
                      cuda_device, nccl_unique_id, rank, nranks, cuda_stream, nullptr);
}

static igs_status create_ctx(igs_ctx** out, int64_t n_global, int64_t row_begin,
                             int64_t n_local, const int64_t* rowptr, const void* colind,
                             int colind_bits, const double* values, int64_t nnz_local,
                             igs_mem where, int cuda_device, const void* nccl_unique_id,
                             int rank, int nranks, void* cuda_stream, const VirtPlan* vp) {
    *out = nullptr;
    ARG_CHECK(n_global > 0, "igs_create: n_global must be > 0");
    ARG_CHECK(row_begin >= 0 && n_local >= 0 && row_begin + n_local <= n_global, "igs_create: bad row block");
    ARG_CHECK(colind_bits == 32 || colind_bits == 64, "igs_create: colind_bits must be 32 or 64");
    ARG_CHECK(nranks >= 1 && rank >= 0 && rank < nranks, "igs_create: bad rank/nranks");
    ARG_CHECK(nnz_local >= 0, "igs_create: nnz_local < 0");
    ARG_CHECK(n_local == 0 || (rowptr && (nnz_local == 0 || (colind && values))), "igs_create: NULL CSR array");
    ARG_CHECK(where == IGS_MEM_HOST || where == IGS_MEM_DEVICE, "igs_create: bad memory kind");
    ARG_CHECK(colind_bits == 64 || n_global < ((int64_t)1 << 31), "igs_create: 32-bit columns need n_global < 2^31");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error("igs_create: no CUDA device (libigs has no CPU fallback)");
        return IGS_ERR_CUDA;
    }
    ARG_CHECK(cuda_device >= 0 && cuda_device < ndev, "igs_create: bad cuda_device");
    CUDA_TRY(cudaSetDevice(cuda_device));

    // host views of the CSR (copy from the device when given device pointers)
    std::vector<int64_t> h_rowptr;
    std::vector<char> h_col;
    std::vector<double> h_val;
    const size_t cbytes = (size_t)nnz_local * (colind_bits / 8);
    if (where == IGS_MEM_DEVICE) {
        h_rowptr.resize(n_local + 1);
        h_col.resize(cbytes);
        h_val.resize(nnz_local);
        if (n_local > 0) CUDA_TRY(cudaMemcpy(h_rowptr.data(), rowptr, sizeof(int64_t) * (n_local + 1), cudaMemcpyDeviceToHost));
        else h_rowptr[0] = 0;
        if (nnz_local) {
            CUDA_TRY(cudaMemcpy(h_col.data(), colind, cbytes, cudaMemcpyDeviceToHost));
            CUDA_TRY(cudaMemcpy(h_val.data(), values, sizeof(double) * nnz_local, cudaMemcpyDeviceToHost));
        }
        rowptr = h_rowptr.data();
        colind = h_col.data();
        values = h_val.data();
    }
    int64_t zero_ptr = 0;
    if (n_local == 0) rowptr = &zero_ptr;
    TRY(validate_csr(n_global, n_local, rowptr, colind, colind_bits, values, nnz_local));

    igs_ctx* ctx = new igs_ctx();
    ctx->dev = cuda_device;
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->n_global = n_global;
    ctx->row_begin = row_begin;
    ctx->n_local = n_local;
    ctx->ldv = round_up(std::max<int64_t>(n_local, 1), 32);
    ctx->nnz = nnz_local;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);

    auto fail = [&](igs_status s) { free_ctx(ctx); return s; };
    if (const char* e = std::getenv("IGS_NCCL_TIMEOUT_S")) ctx->timeout_s = std::max(1e-6, std::atof(e));
    // the fused block dot + NVLink exchange is the G > 1 default (IGS_XCHG=0: a separate
    // ncclAllReduce after each block dot; IGS_XCHG=1 also on one GPU, via a 1-rank comm)
    ctx->xchg_req = nranks > 1 && !vp;
    if (const char* e = std::getenv("IGS_XCHG")) ctx->xchg_req = !vp && std::atoi(e) != 0;
    if (const char* e = std::getenv("IGS_FORCE_NCCL")) ctx->force_nccl = nranks == 1 && std::atoi(e) != 0;
    if (!vp && (nranks > 1 || ctx->xchg_req || ctx->force_nccl)) {
        // (one rank + IGS_XCHG=1: a 1-rank communicator, so the fused exchange path runs on
        //  a single GPU exactly as it does on G)
        ncclUniqueId id;
        if (nranks > 1) std::memcpy(&id, nccl_unique_id, sizeof(id));
        else if (ncclGetUniqueId(&id) != ncclSuccess) {
            set_error("ncclGetUniqueId failed");
            return fail(IGS_ERR_NCCL);
        }
        ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            ctx->comm = nullptr;
            set_error(std::string("ncclCommInitRank failed: ") + ncclGetErrorString(r));
            return fail(IGS_ERR_NCCL);
        }
        if (cudaMalloc(&ctx->d_misc, 2 * sizeof(int)) != cudaSuccess ||
            cudaMemset(ctx->d_misc, 0, 2 * sizeof(int)) != cudaSuccess) {
            set_error("igs_create: cudaMalloc (exchange flags) failed");
            return fail(IGS_ERR_OOM);
        }
        ctx->d_xerr = ctx->d_misc + 1;
    }
    std::vector<int64_t> local_col;
    {
        igs_status s = setup_halo(ctx, rowptr, colind, colind_bits, local_col, vp);
        if (s != IGS_OK) return fail(s);
    }
    // device CSR: int32 rowptr unless nnz needs 64 bits or the caller chose 64-bit columns
    const bool idx64 = colind_bits == 64 || (n_local + ctx->n_ghost) >= ((int64_t)1 << 31);
    const bool ptr64 = idx64 || nnz_local >= ((int64_t)1 << 31);
    ctx->A.nrows = n_local;
    ctx->A.ptr64 = ptr64;
    ctx->A.idx64 = idx64;
    ctx->A.nloc = n_local;
    ctx->A.ghost = ctx->n_ghost > 0 ? ctx->d_ghost : nullptr;
    // short rows (<= 8 nnz on average): CSR-stream kernel (lpr = 0); otherwise vector CSR with
    // lanes per row = next power of two of the mean row length, in [1, 32]
    {
        const double avg = n_local > 0 ? (double)nnz_local / (double)n_local : 1.0;
        int lpr = 1;
        while (lpr < 32 && lpr < avg) lpr *= 2;
        ctx->A.lpr = avg <= 8.0 ? 0 : lpr;
    }
    // SELL-32 copy for short rows (coalesced per-thread rows).  When it exists
    // it is the only full copy of A on the device: the CSR arrays keep just the boundary rows
    // (G > 1: rows with a ghost column, multiplied after the halo by launch_spmv_rows).
    if (n_local <= pcycle_xs_max() && ctx->A.lpr == 32 && nranks == 1) {
        ctx->h_rowlen.resize((size_t)n_local);
        for (int64_t r = 0; r < n_local; r++) ctx->h_rowlen[(size_t)r] = (int32_t)(rowptr[r + 1] - rowptr[r]);
    }
    std::vector<int64_t> bnd;
    {
        const char* es = std::getenv("IGS_SELL");  // test hook: IGS_SELL=0 keeps the CSR kernels
        if (ctx->A.lpr == 0 && n_local > 0 && !(es && std::atoi(es) == 0)) {
            igs_status ss = build_sell(ctx, rowptr, local_col, values, idx64, bnd);
            if (ss != IGS_OK) return fail(ss);
        }
    }
    {
        const bool compact = ctx->A.sell_ptr != nullptr;  // boundary rows only
        const int64_t nr = compact ? (int64_t)bnd.size() : n_local;
        std::vector<int64_t> rpc((size_t)nr + 1, 0);
        for (int64_t i = 0; i < nr; i++) {
            const int64_t r = compact ? bnd[(size_t)i] : i;
            rpc[(size_t)i + 1] = rpc[(size_t)i] + (rowptr[r + 1] - rowptr[r]);
        }
        const int64_t nzc = rpc[(size_t)nr];
        std::vector<char> rp((size_t)(nr + 1) * (ptr64 ? 8 : 4));
        for (int64_t i = 0; i <= nr; i++) {
            if (ptr64) reinterpret_cast<int64_t*>(rp.data())[i] = rpc[(size_t)i];
            else reinterpret_cast<int32_t*>(rp.data())[i] = (int32_t)rpc[(size_t)i];
        }
        std::vector<char> ci((size_t)std::max<int64_t>(nzc, 1) * (idx64 ? 8 : 4));
        std::vector<double> vc;
        const double* vsrc = values;
        if (compact) vc.resize((size_t)std::max<int64_t>(nzc, 1));
        for (int64_t i = 0, at = 0; i < nr; i++) {
            const int64_t r = compact ? bnd[(size_t)i] : i;
            for (int64_t q = rowptr[r]; q < rowptr[r + 1]; q++, at++) {
                if (idx64) reinterpret_cast<int64_t*>(ci.data())[at] = local_col[(size_t)q];
                else reinterpret_cast<int32_t*>(ci.data())[at] = (int32_t)local_col[(size_t)q];
                if (compact) vc[(size_t)at] = values[q];
            }
        }
        if (compact) vsrc = vc.data();
        cudaError_t e;
        const size_t pad = 64;
        if ((e = cudaMalloc(&ctx->d_rowptr, rp.size() + pad)) != cudaSuccess ||
            (e = cudaMalloc(&ctx->d_col, ci.size() + pad)) != cudaSuccess ||
            (e = cudaMalloc(&ctx->d_val, sizeof(double) * std::max<int64_t>(nzc, 1) + pad)) != cudaSuccess ||
            (e = cudaMemset(ctx->d_rowptr, 0, rp.size() + pad)) != cudaSuccess ||
            (e = cudaMemset(ctx->d_col, 0, ci.size() + pad)) != cudaSuccess ||
            (e = cudaMemset(ctx->d_val, 0, sizeof(double) * std::max<int64_t>(nzc, 1) + pad)) != cudaSuccess) {
            set_error(std::string("igs_create: cudaMalloc: ") + cudaGetErrorString(e));
            return fail(IGS_ERR_OOM);
        }
        if ((e = cudaMemcpy(ctx->d_rowptr, rp.data(), rp.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
            (e = cudaMemcpy(ctx->d_col, ci.data(), (size_t)nzc * (idx64 ? 8 : 4), cudaMemcpyHostToDevice)) != cudaSuccess ||
            (e = cudaMemcpy(ctx->d_val, vsrc, sizeof(double) * nzc, cudaMemcpyHostToDevice)) != cudaSuccess) {
            set_error(std::string("igs_create: cudaMemcpy: ") + cudaGetErrorString(e));
            return fail(IGS_ERR_CUDA);
        }
        ctx->csr_compact = compact;
    }
    ctx->A.rowptr = ctx->d_rowptr;
    ctx->A.col = ctx->d_col;
    ctx->A.val = ctx->d_val;
    ctx->bdot_grid = bdot_grid_size(n_local, ctx->num_sms);
    {
        if (const char* e = std::getenv("IGS_GRAPHS")) ctx->graphs_enabled = std::atoi(e) != 0;
        if (const char* e = std::getenv("IGS_PERSIST")) ctx->pc_enabled = std::atoi(e) != 0;
        if (const char* e = std::getenv("IGS_MGS_FUSED")) ctx->mgs_fused = std::atoi(e) != 0;
        if (const char* e = std::getenv("IGS_PC_XSTAGE")) ctx->xs_enabled = std::atoi(e) != 0;
        if (const char* e = std::getenv("IGS_PC_ARES")) ctx->ares_enabled = std::atoi(e) != 0;
        if (const char* e = std::getenv("IGS_TWO_FUSED")) ctx->two_fused = std::atoi(e) != 0;
        if (const char* e = std::getenv("IGS_TWO_FUSED_L2_MB")) ctx->two_fused_l2 = std::atof(e) * 1e6;
        if (const char* e = std::getenv("IGS_PC_NTRI")) ctx->pc_ntri = std::atoi(e);
        if (const char* e = std::getenv("IGS_PC_GRID")) ctx->pc_grid = std::atoi(e);
        if (const char* e = std::getenv("IGS_PC_MAX_N")) ctx->pc_max_n = std::atoll(e);
        if (const char* e = std::getenv("IGS_PC_ROWSPLIT_N")) ctx->pc_rowsplit_n = std::atoll(e);
    }
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_crit, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_tail, cudaEventDisableTiming)) != cudaSuccess) {
        set_error(std::string("igs_create: stream/event: ") + cudaGetErrorString(e));
        return fail(IGS_ERR_CUDA);
    }
    if ((e = cudaMallocHost(&ctx->h_pinned, sizeof(double) * 64)) != cudaSuccess ||
        (e = cudaMallocHost(&ctx->h_pinned_int, sizeof(int) * 64)) != cudaSuccess) {
        set_error(std::string("igs_create: cudaMallocHost: ") + cudaGetErrorString(e));
        return fail(IGS_ERR_OOM);
    }
    ctx->ok = true;
    *out = ctx;
    return IGS_OK;
}

extern "C" igs_status igs_destroy(igs_ctx* ctx) {
    if (!ctx) return IGS_OK;
    cudaSetDevice(ctx->dev);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (VGroup* g = ctx->vgroup) {  // the last member frees the group
        g->members[(size_t)ctx->rank] = nullptr;
        if (--g->alive == 0) delete g;
        ctx->vgroup = nullptr;
    }
    free_ctx(ctx);
    return IGS_OK;
}

// ------------------------------------------------------------------------- workspace
static size_t small_doubles(int m, int k) {
    const size_t ldh = m + 1, dld = 2 * (m + 1) + 2;
    return 3 * ldh * m      // H, HP, R
           + (size_t)m * m  // L
           + 2 * (m + 2)    // cs, sn
           + (m + 2)        // g
           + (m + 1) * dld  // dots
           + 4 * (m + 2)    // alpha, beta, y, gam
           + (m + 3)        // dots2
           + 2 * (size_t)(m + 1) * (m + 2) + (m + 2)  // r1h, r3h, cbd
           + SC_COUNT + 2 * (k + 2);  // res_hist, lnorm
}

extern "C" size_t igs_workspace_bytes(const igs_ctx* ctx, int max_restart) {
    if (!ctx || max_restart < 1) return 0;
    return (size_t)(max_restart + 1) * ctx->ldv * sizeof(double);
}

extern "C" igs_status igs_bind_workspace(igs_ctx* ctx, void* dev_ptr, size_t bytes) {
    ARG_CHECK(ctx && ctx->ok, "igs_bind_workspace: bad context");
    ARG_CHECK(dev_ptr && ((uintptr_t)dev_ptr % 256) == 0, "igs_bind_workspace: pointer must be 256-byte aligned");
    if (ctx->owns_ws && ctx->d_V) { cudaFree(ctx->d_V); }
    ctx->d_V = nullptr;
    ctx->m_cap = 0;
    ctx->bound_ws = dev_ptr;
    ctx->bound_bytes = bytes;
    ctx->owns_ws = false;
    return IGS_OK;
}

// min over ranks of a success flag (every rank takes the same branch afterwards)
static igs_status agree_all(igs_ctx* ctx, bool mine, bool* all) {
    ctx->h_pinned_int[30] = mine ? 1 : 0;
    CUDA_TRY(cudaMemcpyAsync(ctx->d_misc, ctx->h_pinned_int + 30, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    NCCL_TRY(ncclAllReduce(ctx->d_misc, ctx->d_misc, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned_int + 31, ctx->d_misc, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TRY(wait_for(ctx, nullptr, ctx->stream, "fused exchange setup"));
    *all = ctx->h_pinned_int[31] == 1;
    return IGS_OK;
}

static void release_xchg(igs_ctx* ctx) {
    if (ctx->xwin && !ctx->aborted) ncclCommWindowDeregister(ctx->comm, ctx->xwin);
    ctx->xwin = nullptr;
    if (ctx->xbuf && !ctx->aborted) ncclMemFree(ctx->xbuf);
    ctx->xbuf = nullptr;
    cudaFree(ctx->d_xchg);
    ctx->d_xchg = nullptr;
    ctx->xslot = 0;
}

// Symmetric window (2 slots x `slot` doubles + one inbox word per rank, xchg.cuh) and the
// device communicator.  Collective: ensure_workspace runs on every rank in step.  Every
// step that can fail on one rank only (allocation, registration) is followed by an
// agreement allreduce, so either all ranks use the fused exchange or all fall back to
// ncclAllReduce -- a rank that fell back alone would strand its peers at the barrier.
static igs_status setup_xchg(igs_ctx* ctx, int slot, bool* ok_out) {
    *ok_out = true;
    if (ctx->d_xchg && slot <= ctx->xslot) return IGS_OK;
    release_xchg(ctx);
    const size_t inbox_off = (size_t)round_up((int64_t)2 * slot * sizeof(double), 16);
    size_t bytes = inbox_off + sizeof(unsigned) * (size_t)ctx->nranks;
    bytes = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    bool ok = ncclMemAlloc(&ctx->xbuf, bytes) == ncclSuccess;
    if (!ok) ctx->xbuf = nullptr;
    // zero the inboxes before any peer can write into them (the agreement below orders it)
    if (ok) ok = cudaMemsetAsync(ctx->xbuf, 0, bytes, ctx->stream) == cudaSuccess &&
                 cudaStreamSynchronize(ctx->stream) == cudaSuccess;
    bool all = false;
    TRY(agree_all(ctx, ok, &all));
    if (all) {
        ok = ncclCommWindowRegister(ctx->comm, ctx->xbuf, bytes, &ctx->xwin, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess;
        if (!ok) ctx->xwin = nullptr;
        TRY(agree_all(ctx, ok, &all));
    }
    if (all && !ctx->dcomm_ok) {
        ncclDevCommRequirements reqs;
        std::memset(&reqs, 0, sizeof(reqs));
        reqs.lsaBarrierCount = 1;
        ok = ncclDevCommCreate(ctx->comm, &reqs, &ctx->dcomm) == ncclSuccess;
        ctx->dcomm_ok = ok;
        TRY(agree_all(ctx, ok, &all));
    }
    // one NVLink (LSA) domain spanning the communicator: the same on every rank
    if (all) all = ctx->dcomm.lsaSize == ctx->nranks;
    if (all && !ctx->d_xchg) {
        ok = cudaMalloc(&ctx->d_xchg, sizeof(XchgDev) + 16) == cudaSuccess &&
             cudaMemset(ctx->d_xchg, 0, sizeof(XchgDev) + 16) == cudaSuccess;
        if (!ok) ctx->d_xchg = nullptr;
        TRY(agree_all(ctx, ok, &all));
    }
    if (!all) {
        release_xchg(ctx);
        *ok_out = false;
        return IGS_OK;
    }
    XchgDev& h = ctx->h_xchg;
    std::memset(&h, 0, sizeof(h));
    h.comm = ctx->dcomm;
    h.win = ctx->xwin;
    h.calls = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ctx->d_xchg) + sizeof(XchgDev));
    h.err = ctx->d_xerr;
    h.timeout_ns = (unsigned long long)(ctx->timeout_s * 1e9);
    h.stall_call = 0xffffffffu;
    if (const char* e = std::getenv("IGS_TEST_XCHG_STALL")) h.stall_call = (unsigned)std::atoi(e);  // test hook
    h.slot_doubles = slot;
    h.nranks = ctx->nranks;
    h.me = ctx->dcomm.lsaRank;
    h.inbox_off = inbox_off;
    CUDA_TRY(cudaMemcpy(ctx->d_xchg, &h, sizeof(h), cudaMemcpyHostToDevice));
    ctx->xslot = slot;
    return IGS_OK;
}

static igs_status ensure_workspace(igs_ctx* ctx, int m, int k, bool host_vec) {
    const int64_t ldv = ctx->ldv;
    if (m > ctx->m_cap || k > ctx->k_cap) {
        const int mm = std::max(m, ctx->m_cap), kk = std::max(k, ctx->k_cap);
        // V
        const size_t vbytes = (size_t)(mm + 1) * ldv * sizeof(double);
        if (ctx->owns_ws) {
            cudaFree(ctx->d_V);
            ctx->d_V = nullptr;
            CUDA_TRY(cudaMalloc(&ctx->d_V, vbytes));
        } else {
            if (vbytes > ctx->bound_bytes) {
                set_error("igs_solve: bound workspace too small");
                return IGS_ERR_OOM;
            }
            ctx->d_V = static_cast<double*>(ctx->bound_ws);
        }
        for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);
        ctx->graphs.clear();
        // zero once: padding rows of every column must stay 0 (kernels read them as 0)
        CUDA_TRY(cudaMemsetAsync(ctx->d_V, 0, vbytes, ctx->stream));
        cudaFree(ctx->d_small);
        cudaFree(ctx->d_int);
        cudaFree(ctx->d_part);
        const size_t nsd = small_doubles(mm, kk);
        CUDA_TRY(cudaMalloc(&ctx->d_small, nsd * sizeof(double)));
        CUDA_TRY(cudaMemsetAsync(ctx->d_small, 0, nsd * sizeof(double), ctx->stream));
        CUDA_TRY(cudaMalloc(&ctx->d_int, sizeof(int) * ST_COUNT));
        CUDA_TRY(cudaMemsetAsync(ctx->d_int, 0, sizeof(int) * ST_COUNT, ctx->stream));
        // rows of partials: any reduction kernel's grid (block dots, the persistent kernel's
        // row-block dots with up to one CTA per SM)
        ctx->part_rows = std::max(ctx->bdot_grid, ctx->num_sms);
        CUDA_TRY(cudaMalloc(&ctx->d_part, sizeof(double) * (size_t)ctx->part_rows * (2 * (mm + 1) + 2)));
        Dev& d = ctx->dev_state;
        d.m = mm;
        d.ldh = mm + 1;
        d.dld = 2 * (mm + 1) + 2;
        double* q = ctx->d_small;
        auto take = [&](size_t cnt) { double* r = q; q += cnt; return r; };
        d.H = take((size_t)d.ldh * mm);
        d.HP = take((size_t)d.ldh * mm);
        d.R = take((size_t)d.ldh * mm);
        d.L = take((size_t)mm * mm);
        d.cs = take(mm + 2);
        d.sn = take(mm + 2);
        d.g = take(mm + 2);
        d.dots = take((size_t)(mm + 1) * d.dld);
        d.alpha = take(mm + 2);
        d.beta = take(mm + 2);
        d.y = take(mm + 2);
        d.gam = take(mm + 2);
        d.dots2 = take(mm + 3);
        d.r1h = take((size_t)(mm + 1) * (mm + 2));
        d.r3h = take((size_t)(mm + 1) * (mm + 2));
        d.cbd = take(mm + 2);
        d.scal = take(SC_COUNT);
        d.res_hist = take(kk + 2);
        d.lnorm = take(kk + 2);
        d.istate = ctx->d_int;
        ctx->m_cap = mm;
        ctx->k_cap = kk;
        if (ctx->xchg_req) {
            bool ok = true;
            TRY(setup_xchg(ctx, d.dld, &ok));
            if (!ok) {  // on every rank (agreed): keep ncclAllReduce
                std::fprintf(stderr, "[igs] fused NVLink exchange unavailable on some rank; using ncclAllReduce\n");
                ctx->xchg_req = false;
            }
        }
    }
    if (!ctx->d_z) {
        CUDA_TRY(cudaMalloc(&ctx->d_z, sizeof(double) * ldv));
        CUDA_TRY(cudaMemsetAsync(ctx->d_z, 0, sizeof(double) * ldv, ctx->stream));
    }
    if (!ctx->d_counter) {
        CUDA_TRY(cudaMalloc(&ctx->d_counter, sizeof(unsigned) * 12));  // [4..11]: persistent-kernel flags
        CUDA_TRY(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned) * 12, ctx->stream));
    }
    if (host_vec && !ctx->d_b) {
        CUDA_TRY(cudaMalloc(&ctx->d_b, sizeof(double) * ldv));
        CUDA_TRY(cudaMalloc(&ctx->d_x, sizeof(double) * ldv));
        CUDA_TRY(cudaMemsetAsync(ctx->d_b, 0, sizeof(double) * ldv, ctx->stream));
        CUDA_TRY(cudaMemsetAsync(ctx->d_x, 0, sizeof(double) * ldv, ctx->stream));
    }
    return IGS_OK;
}

// -------------------------------------------------------------------- solve pieces
static inline double* Vcol(igs_ctx* c, int j) { return c->d_V + (int64_t)j * c->ldv; }

static double spmv_bytes(const igs_ctx* c) {
    const double sc = c->A.idx64 ? 8 : 4, sp = c->A.ptr64 ? 8 : 4;
    return (double)c->nnz * (8 + sc) + (double)(c->n_local + 1) * sp + 16.0 * c->n_local +
           8.0 * c->n_ghost;
}

// igs_virtual_solve's allreduce: every member stages its vector (call parity slot), meets
// the others at the host barrier, then sums the G slots in member order into its own
// buffer after cross-stream waits on the peers' staging copies -- the same order on every
// member, so the replicated small state stays bitwise identical, as with NCCL.  A slot is
// rewritten two calls later only after every member's sum that read it (events).
static igs_status vallreduce(igs_ctx* ctx, double* buf, int64_t count) {
    VGroup& g = *ctx->vgroup;
    const int r = ctx->rank, G = g.G;
    const uint64_t call = ctx->v_ar_calls++;
    const int par = (int)(call & 1);
    ARG_CHECK((size_t)count <= ctx->vstage_cap, "virtual allreduce: staging slot too small");
    cudaStream_t st = ctx->stream;
    if (call >= 2)
        for (int q = 0; q < G; q++) CUDA_TRY(cudaStreamWaitEvent(st, g.ev_sum[par][q], 0));
    double* slot = ctx->d_vstage + (size_t)par * ctx->vstage_cap;
    CUDA_TRY(cudaMemcpyAsync(slot, buf, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaEventRecord(g.ev_copy[par][r], st));
    if (!g.barrier()) {
        set_error("virtual allreduce: a member failed or did not arrive");
        return IGS_ERR_STATE;
    }
    for (int q = 0; q < G; q++) CUDA_TRY(cudaStreamWaitEvent(st, g.ev_copy[par][q], 0));
    launch_rank_sum(g.d_stage_ptrs + (size_t)par * G, G, count, buf, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(g.ev_sum[par][r], st));
    ctx->n_allreduce++;
    return IGS_OK;
}

static igs_status allreduce(igs_ctx* ctx, double* buf, int64_t count) {
    if (ctx->vsolve) return vallreduce(ctx, buf, count);
    if (ctx->nranks == 1 && !ctx->force_nccl) return IGS_OK;
    TIMED(IGS_K_ALLREDUCE, 0.0,
          { NCCL_TRY(ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, ctx->comm, ctx->stream)); });
    ctx->n_allreduce++;
    return IGS_OK;
}

// igs_virtual_solve's halo: barrier A (every member has enqueued its ghost copies of the
// previous exchange), pack once the peers' copies out of this member's send buffer are done,
// barrier B (every member has packed), then this member's ghost copies from the owners' send
// buffers after cross-stream waits on their pack events.  Every member takes part even with
// no peers (the barriers count calls).
static igs_status vhalo(igs_ctx* ctx, const double* x, const int* istate, cudaStream_t st) {
    VGroup& g = *ctx->vgroup;
    const int r = ctx->rank;
    ctx->v_halo_calls++;
    if (!g.barrier()) {
        set_error("virtual halo: a member failed or did not arrive");
        return IGS_ERR_STATE;
    }
    for (size_t i = 0; i < ctx->peers.size(); i++)
        if (ctx->send_cnt[i]) CUDA_TRY(cudaStreamWaitEvent(st, g.ev_hcopy[(size_t)ctx->peers[i]], 0));
    launch_pack(ctx->n_send, ctx->d_send_idx, x, ctx->d_send, istate, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(g.ev_pack[(size_t)r], st));
    if (!g.barrier()) {
        set_error("virtual halo: a member failed or did not arrive");
        return IGS_ERR_STATE;
    }
    for (size_t i = 0; i < ctx->peers.size(); i++) {
        if (!ctx->recv_cnt[i]) continue;
        const igs_ctx* q = g.members[(size_t)ctx->peers[i]];
        const size_t j = (size_t)(std::find(q->peers.begin(), q->peers.end(), ctx->rank) - q->peers.begin());
        ARG_CHECK(j < q->peers.size() && q->send_cnt[j] == ctx->recv_cnt[i], "virtual halo: inconsistent plan");
        CUDA_TRY(cudaStreamWaitEvent(st, g.ev_pack[(size_t)ctx->peers[i]], 0));
        CUDA_TRY(cudaMemcpyAsync(ctx->d_ghost + ctx->recv_off[i], q->d_send + q->send_off[j],
                                 sizeof(double) * ctx->recv_cnt[i], cudaMemcpyDeviceToDevice, st));
    }
    CUDA_TRY(cudaEventRecord(g.ev_hcopy[(size_t)r], st));
    ctx->n_halo += (int64_t)ctx->peers.size();
    return IGS_OK;
}

static igs_status halo_on(igs_ctx* ctx, const double* x, const int* istate, cudaStream_t st) {
    if (ctx->vsolve) return vhalo(ctx, x, istate, st);
    if (ctx->vgroup) {
        // virtual ranks (test hook): the ghosts come from the owners' send buffers, which
        // igs_virtual_spmv packed (pack kernel) before any rank's SpMV was enqueued
        for (size_t i = 0; i < ctx->peers.size(); i++) {
            if (!ctx->recv_cnt[i]) continue;
            const igs_ctx* q = ctx->vgroup->members[(size_t)ctx->peers[i]];
            const size_t j = (size_t)(std::find(q->peers.begin(), q->peers.end(), ctx->rank) - q->peers.begin());
            ARG_CHECK(j < q->peers.size() && q->send_cnt[j] == ctx->recv_cnt[i], "virtual halo: inconsistent plan");
            CUDA_TRY(cudaMemcpyAsync(ctx->d_ghost + ctx->recv_off[i], q->d_send + q->send_off[j],
                                     sizeof(double) * ctx->recv_cnt[i], cudaMemcpyDeviceToDevice, st));
        }
        ctx->n_halo += (int64_t)ctx->peers.size();
        return IGS_OK;
    }
    launch_pack(ctx->n_send, ctx->d_send_idx, x, ctx->d_send, istate, st);
    NCCL_TRY(ncclGroupStart());
    for (size_t i = 0; i < ctx->peers.size(); i++) {
        if (ctx->send_cnt[i]) NCCL_TRY(ncclSend(ctx->d_send + ctx->send_off[i], ctx->send_cnt[i], ncclDouble, ctx->peers[i], ctx->comm, st));
        if (ctx->recv_cnt[i]) NCCL_TRY(ncclRecv(ctx->d_ghost + ctx->recv_off[i], ctx->recv_cnt[i], ncclDouble, ctx->peers[i], ctx->comm, st));
    }
    NCCL_TRY(ncclGroupEnd());
    ctx->n_halo += (int64_t)ctx->peers.size();
    return IGS_OK;
}

static igs_status halo(igs_ctx* ctx, const double* x, const int* istate) {
    if ((ctx->nranks == 1 || ctx->peers.empty()) && !ctx->vsolve) return IGS_OK;
    TIMED(IGS_K_HALO, 16.0 * ctx->n_send + 8.0 * ctx->n_ghost, { TRY(halo_on(ctx, x, istate, ctx->stream)); });
    return IGS_OK;
}

// z = A x (with halo) ; resid: y = b - A x.  G > 1 with SELL: the halo runs on its own
// stream while the interior rows (no ghost column) are multiplied; the boundary rows follow
// once the ghosts have arrived (halo overlapped with the interior SpMV).
static igs_status spmv(igs_ctx* ctx, const double* x, double* y, const double* b, bool resid,
                       const int* istate, int kind) {
    const double by = spmv_bytes(ctx) + (resid ? 8.0 * ctx->n_local : 0.0);
    if (ctx->A.n_bnd > 0 && ctx->hstream) {
        CUDA_TRY(cudaEventRecord(ctx->ev_x, ctx->stream));
        CUDA_TRY(cudaStreamWaitEvent(ctx->hstream, ctx->ev_x, 0));
        if (!ctx->peers.empty() || ctx->vsolve) TRY(halo_on(ctx, x, istate, ctx->hstream));
        CUDA_TRY(cudaEventRecord(ctx->ev_h, ctx->hstream));
        TIMED(kind, by, {
            launch_spmv(ctx->A, x, y, b, resid, istate, ctx->stream);            // interior rows
            CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_h, 0));
            launch_spmv_rows(ctx->A, x, y, b, resid, istate, ctx->stream);       // boundary rows
        });
        return IGS_OK;
    }
    TRY(halo(ctx, x, istate));
    TIMED(kind, by, launch_spmv(ctx->A, x, y, b, resid, istate, ctx->stream));
    return IGS_OK;
}

static igs_status bdot(igs_ctx* ctx, int p, const double* u, const double* z, double* out,
                       const int* istate, int kind) {
    const double by = 8.0 * ctx->n_local * (p + 1 + (z ? 1 : 0));
    if (ctx->d_xchg) {
        // block dot with the cross-rank sum fused in.  The kernel joins the exchange on every
        // rank even when this rank's status word says the cycle has stopped (it then skips the
        // work only): the status word is written by the side-stream tail and can differ
        // between ranks for an iteration or two, so no wait on the tail is needed here.
        TIMED(kind, by,
              launch_block_dot(ctx->n_local, p, ctx->d_V, ctx->ldv, u, z, out, ctx->d_part,
                               ctx->d_counter, ctx->bdot_grid, istate, ctx->stream, ctx->d_xchg));
        ctx->n_allreduce++;
        ctx->n_reduce++;
        return IGS_OK;
    }
    TIMED(kind, by,
          launch_block_dot(ctx->n_local, p, ctx->d_V, ctx->ldv, u, z, out, ctx->d_part,
                           ctx->d_counter, ctx->bdot_grid, istate, ctx->stream));
    TRY(allreduce(ctx, out, z ? 2 * (p + 1) : p + 1));
    ctx->n_reduce++;
    return IGS_OK;
}

// Scalar D2H through pinned staging (synchronises the stream).
static igs_status fetch(igs_ctx* ctx, const double* dsrc, int nd, double* hd, const int* isrc,
                        int ni, int* hi) {
    if (nd) CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned, dsrc, sizeof(double) * nd, cudaMemcpyDeviceToHost, ctx->stream));
    if (ni) CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned_int, isrc, sizeof(int) * ni, cudaMemcpyDeviceToHost, ctx->stream));
    TRY(wait_for(ctx, nullptr, ctx->stream, "igs_solve"));
    if (nd) std::memcpy(hd, ctx->h_pinned, sizeof(double) * nd);
    if (ni) std::memcpy(hi, ctx->h_pinned_int, sizeof(int) * ni);
    return IGS_OK;
}

// One restart cycle of m iterations (SURVEY §8(c) "Cycle priming" + per-iteration body).
// On entry z holds r = b - A x and dots[0] = ||r||^2.  Returns after enqueueing (and occasionally waiting at
// checkpoints, identically on every rank).
static igs_status run_cycle_mgs(igs_ctx* ctx, int m, int t0);

// alg: IGS_ALG_IGS1 (1), IGS_ALG_IGS2 (2, Alg. 3), IGS_ALG_IGS2_TWO (3, Alg. 2 literal),
// IGS_ALG_MGS (4).  Algorithms 1 and 3 share the gs = 1 small-step stages.
static bool use_pcycle(const igs_ctx* ctx, int alg) {
    return ctx->pc_enabled && ctx->nranks == 1 && !ctx->xchg_req && !ctx->force_nccl && ctx->A.n_bnd == 0 &&
           ctx->n_local <= (ctx->pc_max_n >= 0 ? ctx->pc_max_n : (alg == IGS_ALG_IGS2 ? 210000 : 120000)) &&
           (alg == IGS_ALG_IGS1 || alg == IGS_ALG_IGS2) && ctx->dev_state.m <= 1024;
}

static igs_status run_cycle(igs_ctx* ctx, int m, int alg, int t0) {
    if (alg == IGS_ALG_MGS) return run_cycle_mgs(ctx, m, t0);
    const int gs = alg == IGS_ALG_IGS2 ? 2 : 1;
    const bool two_reduce = alg == IGS_ALG_IGS2_TWO;
    Dev& d = ctx->dev_state;
    cudaStream_t st = ctx->stream;
    const int64_t n = ctx->n_local;
    const int* ist = d.istate;
    CUDA_TRY(cudaMemsetAsync(d.H, 0, sizeof(double) * (size_t)d.ldh * d.m, st));
    // priming, Steps 1-2 (reading R2): rho, v_0 = r/rho.  ||r||^2 is already in
    // dots[0] (reduced by igs_solve for the cycle-start residual test).
    TIMED(IGS_K_SMALL, 0.0, launch_small(d, SS_PRIME_NORM, gs, 0, m, t0, st));
    TIMED(IGS_K_UPDATE, 16.0 * n,
          launch_update(n, 0, ctx->d_V, ctx->ldv, ctx->d_z, nullptr, nullptr, nullptr,
                        d.scal + SC_GAMMA, Vcol(ctx, 0), nullptr, ist, 0, st));
    // z = A v_0 ; h = v_0 . z ; u = z - h v_0
    TRY(spmv(ctx, Vcol(ctx, 0), ctx->d_z, nullptr, false, ist, IGS_K_SPMV));
    TRY(bdot(ctx, 0, Vcol(ctx, 0), ctx->d_z, d.dots, ist, IGS_K_BLOCK_DOT));
    TIMED(IGS_K_SMALL, 0.0, launch_small(d, SS_PRIME_H, gs, 0, m, t0, st));
    TIMED(IGS_K_UPDATE, 24.0 * n,
          launch_update(n, 0, ctx->d_V, ctx->ldv, Vcol(ctx, 0), ctx->d_z, nullptr, d.beta,
                        d.scal + SC_GAMMA, Vcol(ctx, 0), Vcol(ctx, 1), ist, 0, st));

    if (use_pcycle(ctx, alg)) {
        // iterations 1..m in one cooperative launch; grid sized so every CTA has >= 64 KB of
        // the iteration's bytes (CSR + V), at most one CTA per SM
        const double iter_bytes = spmv_bytes(ctx) + 8.0 * n * (m + 1);
        int grid = ctx->pc_grid > 0 ? ctx->pc_grid : (int)std::ceil(iter_bytes / 32768.0) + 1;
        grid = std::max(1, std::min(grid, ctx->num_sms));
        CUDA_TRY(cudaMemsetAsync(ctx->d_counter + 4, 0, 8 * sizeof(unsigned), st));
        if (std::getenv("IGS_PC_PROF") && !ctx->d_pcprof) {
            CUDA_TRY(cudaMalloc(&ctx->d_pcprof, sizeof(unsigned long long) * 24 * (size_t)(ctx->dev_state.m + 2)));
        }
        if (ctx->d_pcprof)
            CUDA_TRY(cudaMemsetAsync(ctx->d_pcprof, 0, sizeof(unsigned long long) * 24 * (size_t)(ctx->dev_state.m + 2), st));
        const double by = (double)m * spmv_bytes(ctx) + 16.0 * n * 0.5 * m * (m + 1);
        TIMED(IGS_K_PERSIST, by, {
            // row-block dots above pc_rowsplit_n rows (each CTA would otherwise re-read u, z)
            // (round 1 also required grid - 1 <= bdot_grid, the partials' old capacity: n = 90000
            //  and 147456 fell back to whole-column dots at 0.37-0.47x the graph path's speed)
            double* part = (n >= ctx->pc_rowsplit_n && grid - 1 <= ctx->part_rows) ? ctx->d_part : nullptr;
            // long rows on the CSR phase (no SELL copy): stage u in shared memory
            const int xs = ctx->xs_enabled && !ctx->A.sell_ptr && n <= pcycle_xs_max() &&
                           ctx->nnz >= 32 * n;
            // two forward-substitution CTAs on alternate iterations once the order-p solve
            // outlasts an iteration (long cycles)
            const int ntri = ctx->pc_ntri > 0 ? ctx->pc_ntri : (m >= 128 && grid >= 8 ? 2 : 1);
            // long rows with u staged: keep A itself in shared memory for the cycle when every
            // worker CTA's rows fit (c2: 24 MB of CSR over 145 CTAs); the launcher drops it
            // when they do not
            int ares = 0;
            if (xs && ctx->ares_enabled && !ctx->h_rowlen.empty()) {
                const int W = pcycle_worker_ctas(grid, gs, ntri);
                std::vector<int64_t> per((size_t)W, 0);
                for (int64_t r = 0; r < n; r++) per[(size_t)(r % W)] += ctx->h_rowlen[(size_t)r];
                ares = (int)std::min<int64_t>(*std::max_element(per.begin(), per.end()), INT32_MAX);
            }
            cudaError_t el_ = launch_pcycle(d, ctx->A, ctx->d_V, ctx->ldv, ctx->d_z, n, m, gs,
                                           ctx->d_counter + 4, ctx->d_counter, grid, st, ctx->d_pcprof, part, xs,
                                           ntri, &ares);
            ctx->last_ares = ares;
            CUDA_TRY(el_);
        });
        if (ctx->d_pcprof) {  // IGS_PC_PROF=1: mean phase durations of this cycle to stderr
            std::vector<unsigned long long> pr((size_t)(m + 2) * 24);
            CUDA_TRY(cudaMemcpyAsync(pr.data(), ctx->d_pcprof, pr.size() * 8, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            double acc[8] = {0};
            int cnt = 0;
            for (int p = 2; p < m; p++) {
                const unsigned long long* q = pr.data() + (size_t)p * 8;
                const unsigned long long* qn = pr.data() + (size_t)(p + 1) * 8;
                if (!q[0] || !qn[0]) continue;
                acc[0] += q[1] - q[0]; acc[1] += q[2] - q[1]; acc[2] += q[3] - q[2]; acc[3] += q[4] - q[3];
                acc[4] += q[5] - q[4]; acc[5] += qn[0] - q[5]; acc[6] += q[7] - q[6]; acc[7] += qn[0] - q[0];
                cnt++;
            }
            if (cnt)
                std::fprintf(stderr, "[pcycle grid=%d m=%d] us/iter: A+bar %.2f  B+bar %.2f  C %.2f  bar %.2f  D %.2f  bar %.2f  | tail %.2f | total %.2f\n",
                             grid, m, acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3, acc[3] / cnt / 1e3,
                             acc[4] / cnt / 1e3, acc[5] / cnt / 1e3, acc[6] / cnt / 1e3, acc[7] / cnt / 1e3);
            {  // tail sub-steps (Alg. 3): H column | Givens | status | L row + Step 15 GEMV | hp store
                double t[6] = {0};
                int c2 = 0;
                for (int p = 2; p < m; p++) {
                    const unsigned long long* q = pr.data() + (size_t)(m + 2) * 8 + (size_t)p * 8;
                    const unsigned long long* q0 = pr.data() + (size_t)p * 8;
                    if (!q[0] || !q[5] || !q[6]) continue;
                    for (int k = 0; k < 5; k++) t[k] += (double)(q[k + 1] - q[k]);
                    t[5] += (double)(q[6] - q0[2]);
                    c2++;
                }
                double cr[3] = {0};
                int c3n = 0;
                for (int p = 2; p < m; p++) {  // Alg. 2 one sweep, CTA 0's critical step
                    const unsigned long long* q = pr.data() + (size_t)(m + 2) * 16 + (size_t)p * 8;
                    if (!q[0] || !q[3]) continue;
                    for (int k = 0; k < 3; k++) cr[k] += (double)(q[k + 1] - q[k]);
                    c3n++;
                }
                if (c3n)
                    std::fprintf(stderr, "[pcycle crit] us/iter: pre %.2f  trisolve %.2f  post %.2f\n",
                                 cr[0] / c3n / 1e3, cr[1] / c3n / 1e3, cr[2] / c3n / 1e3);
                if (c2)
                    std::fprintf(stderr, "[pcycle tail] us/iter: Hcol %.2f  givens %.2f  status %.2f  GEMV %.2f  hp %.2f | C wait %.2f\n",
                                 t[0] / c2 / 1e3, t[1] / c2 / 1e3, t[2] / c2 / 1e3, t[3] / c2 / 1e3, t[4] / c2 / 1e3,
                                 t[5] / c2 / 1e3);
            }
        }
        ctx->n_pcycle++;
        ctx->n_iter += m;
        ctx->n_reduce += m;
        if (!ctx->capturing) TRY(wait_for(ctx, nullptr, st, "igs_solve: cycle"));
        return IGS_OK;
    }
    const int poll_every = 16;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int ev_slot = 0, ev_pending = -1;
    int* h_status = ctx->h_pinned_int + 16;  // 2 slots
    for (int p = 1; p <= m; p++) {
        const bool drain = (p == m);
        double* u = Vcol(ctx, p);
        if (!drain) TRY(spmv(ctx, u, ctx->d_z, nullptr, false, ist, IGS_K_SPMV));  // Step 4
        TRY(bdot(ctx, p, u, drain ? nullptr : ctx->d_z, d.dots + (int64_t)p * d.dld, ist, IGS_K_BLOCK_DOT));
        // (no wait on tail(p-1): the critical step reads nothing the tail writes; a stop the
        //  tail decides is seen one iteration later at worst, and the tails stay ordered on
        //  the side stream; the cycle end joins the side stream)
        TIMED(IGS_K_SMALL, 0.0, launch_small(d, SS_CRIT, gs, p, m, t0, st));
        // tail of the small step on the side stream, overlapped with the fused update
        CUDA_TRY(cudaEventRecord(ctx->ev_crit, st));
        CUDA_TRY(cudaStreamWaitEvent(ctx->side, ctx->ev_crit, 0));
        // (untimed: its events would span the concurrent update; counted as a launch)
        launch_small(d, SS_TAIL, gs, p, m, t0, ctx->side);
        CUDA_TRY(cudaGetLastError());
        if (ctx->timing) ctx->tail_launches++;
        CUDA_TRY(cudaEventRecord(ctx->ev_tail, ctx->side));
        {
            const double ub = 8.0 * n * ((gs == 2 || !drain) ? p : 0) + 16.0 * n + (drain ? 0.0 : 16.0 * n);
            // the dots re-read the CTAs' tiles from L2: fused while grid x 512 rows x p
            // columns stays within ~80 MB (p <= 32 at 4 CTAs per SM; measured slower beyond)
            // shared-memory tile variant (bulk copies) while two R x (p + 2) tiles fit (p <= ~103)
            // (the L2 re-read variant is faster while its tiles fit in L2: small p first)
            // (small n: the separate block dot spreads the columns over more CTAs -- c2 was
            // 7.6K vs 9.6K it/s fused -- so fuse only with at least one 512-row tile per SM)
            const bool fuse2_l2 = two_reduce && !drain && ctx->two_fused && n >= (int64_t)ctx->num_sms * 512 &&
                                  (double)update_dot_grid(n, ctx->num_sms) * 512.0 * p * 8.0 <= ctx->two_fused_l2;
            const bool fuse2_tma = !fuse2_l2 && two_reduce && !drain && ctx->two_fused && p >= 1 &&
                                   n >= (int64_t)ctx->num_sms * 512 &&
                                   update_dot_tma_rows(p) > 0 && (ctx->ldv % 2) == 0 &&
                                   ((uintptr_t)ctx->d_V % 16) == 0 && ((uintptr_t)u % 16) == 0 &&
                                   ((uintptr_t)ctx->d_z % 16) == 0;
            const bool fuse2 = fuse2_tma || fuse2_l2;
            if (fuse2) {
                // Alg. 2 two-reduce: the update fused with the second sweep's block dot
                // r2 = V_{p+1}^T u' (one HBM read of V_p; the dots re-read it from L2)
                const int64_t ntl = fuse2_tma ? (n + update_dot_tma_rows(p) - 1) / update_dot_tma_rows(p) : 1;
                int grid = fuse2_tma ? (int)std::min<int64_t>(ntl, ctx->num_sms) : update_dot_grid(n, ctx->num_sms);
                const int64_t cap = (int64_t)ctx->bdot_grid * (2 * (d.m + 1) + 2) / (p + 2);
                grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, cap));
                const int* ist2 = ist;  // with the exchange the kernel joins it even when stopped
                if (fuse2_tma)
                    TIMED(IGS_K_UPDATE, ub,
                          launch_update_dot_tma(n, p, ctx->d_V, ctx->ldv, u, ctx->d_z, gs == 2 ? d.alpha : nullptr,
                                                d.beta, d.scal + SC_GAMMA, u, Vcol(ctx, p + 1), ist2, p, ctx->d_part,
                                                d.dots2, ctx->d_counter, grid, ctx->d_xchg, st));
                else
                    TIMED(IGS_K_UPDATE, ub,
                          launch_update_dot(n, p, ctx->d_V, ctx->ldv, u, ctx->d_z, gs == 2 ? d.alpha : nullptr, d.beta,
                                            d.scal + SC_GAMMA, u, Vcol(ctx, p + 1), ist2, p, ctx->d_part, d.dots2,
                                            ctx->d_counter, grid, ctx->d_xchg, st));
                ctx->n_reduce++;
                if (ctx->d_xchg) ctx->n_allreduce++;
                else TRY(allreduce(ctx, d.dots2, p + 2));
            } else {
                TIMED(IGS_K_UPDATE, ub,
                      launch_update(n, p, ctx->d_V, ctx->ldv, u, ctx->d_z, gs == 2 ? d.alpha : nullptr,
                                    d.beta, d.scal + SC_GAMMA, u, drain ? nullptr : Vcol(ctx, p + 1), ist, p, st));
            }
            if (two_reduce && !drain) {
                // Alg. 2 Steps 14-16: r2 = V_{p+1}^T u (second reduction), r3 = (I+L)^{-1} r2,
                // w = u - V_{p+1} r3 (in place), H[:p+1, p] = r1 + r3
                double* un = Vcol(ctx, p + 1);
                if (!fuse2) TRY(bdot(ctx, p + 1, un, nullptr, d.dots2, ist, IGS_K_BLOCK_DOT));
                TIMED(IGS_K_SMALL, 0.0, launch_small(d, SS_CRIT2, gs, p, m, t0, st));
                TIMED(IGS_K_UPDATE, 8.0 * n * (p + 1) + 16.0 * n,
                      launch_update(n, p + 1, ctx->d_V, ctx->ldv, un, nullptr, d.alpha, nullptr,
                                    d.scal + SC_ONE, un, nullptr, ist, p, st));
            }
        }
        ctx->n_iter++;
        // checkpoint: copy the status word; decide on the PREVIOUS checkpoint's value so the
        // GPU always has one chunk queued and every rank stops at the same iteration
        if (!ctx->capturing && p % poll_every == 0 && p < m) {
            if (!ev[0]) {
                CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
                CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
            }
            // with collectives in the loop the copied status must be the same on every rank:
            // read it after tail(p) (the status through iteration p is then final), so all
            // ranks leave the loop at the same checkpoint and issue the same collectives
            if (ctx->comm || ctx->vsolve) CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_tail, 0));
            CUDA_TRY(cudaMemcpyAsync(h_status + ev_slot, ist + ST_STATUS, sizeof(int), cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaEventRecord(ev[ev_slot], st));
            if (ev_pending >= 0) {
                TRY(wait_for(ctx, ev[ev_pending], nullptr, "igs_solve: checkpoint"));
                if (h_status[ev_pending] != RUNNING) { ev_pending = -1; break; }
            }
            ev_pending = ev_slot;
            ev_slot ^= 1;
        }
    }
    CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_tail, 0));
    if (!ctx->capturing) TRY(wait_for(ctx, nullptr, st, "igs_solve: cycle"));
    if (ev[0]) { cudaEventDestroy(ev[0]); cudaEventDestroy(ev[1]); }
    return IGS_OK;
}

// MGS-GMRES cycle (the sync-count baseline): column j needs j+1
// separate inner products and one norm, each a device reduction (+ allreduce when G > 1).
// One fused MGS step (launch_mgs_step): H = *hsrc, w -= *hsrc v (v != NULL), then
// *out = vn . w (vn != NULL) or w . w -- one reduction, summed across ranks like bdot().
static igs_status mgs_step(igs_ctx* ctx, const double* v, const double* vn, const double* hsrc,
                           double* out, double* Hdst) {
    const int64_t n = ctx->n_local;
    const int* ist = ctx->dev_state.istate;
    int grid = mgs_step_grid(n, ctx->num_sms);
    grid = std::min(grid, 4 * ctx->bdot_grid - 1);
    const double by = 8.0 * n * ((v ? 3 : 1) + (vn ? 1 : 0));
    // (with the exchange the kernel joins it even when stopped; see bdot())
    TIMED(IGS_K_BLOCK_DOT, by,
          launch_mgs_step(n, v, ctx->d_z, vn, hsrc, Hdst, ctx->d_part, out, ctx->d_counter, grid, ist,
                          ctx->d_xchg, ctx->stream));
    ctx->n_reduce++;
    if (ctx->d_xchg) {
        ctx->n_allreduce++;
        return IGS_OK;
    }
    return allreduce(ctx, out, 1);
}

static igs_status run_cycle_mgs(igs_ctx* ctx, int m, int t0) {
    Dev& d = ctx->dev_state;
    cudaStream_t st = ctx->stream;
    const int64_t n = ctx->n_local;
    const int* ist = d.istate;
    // fused projection + next dot (default; IGS_MGS_FUSED=0: separate dot and axpy kernels)
    const bool fused = ctx->mgs_fused && ((uintptr_t)ctx->d_z % 16) == 0 && ((uintptr_t)ctx->d_V % 16) == 0 &&
                       (ctx->ldv % 2) == 0;
    CUDA_TRY(cudaMemsetAsync(d.H, 0, sizeof(double) * (size_t)d.ldh * d.m, st));
    TIMED(IGS_K_SMALL, 0.0, launch_small(d, SS_PRIME_NORM, 1, 0, m, t0, st));
    TIMED(IGS_K_UPDATE, 16.0 * n,
          launch_update(n, 0, ctx->d_V, ctx->ldv, ctx->d_z, nullptr, nullptr, nullptr,
                        d.scal + SC_GAMMA, Vcol(ctx, 0), nullptr, ist, 0, st));
    const int poll_every = 16;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int ev_slot = 0, ev_pending = -1;
    int* h_status = ctx->h_pinned_int + 16;
    for (int j = 0; j < m; j++) {
        TRY(spmv(ctx, Vcol(ctx, j), ctx->d_z, nullptr, false, ist, IGS_K_SPMV));
        if (fused) {
            // h_0 = v_0 . w; then projection i fused with the next dot (or ||w||^2 after i = j)
            TRY(mgs_step(ctx, nullptr, Vcol(ctx, 0), nullptr, d.dots + 1, nullptr));
            for (int i = 0; i <= j; i++)
                TRY(mgs_step(ctx, Vcol(ctx, i), i < j ? Vcol(ctx, i + 1) : nullptr, d.dots + 1 + (i & 1),
                             i < j ? d.dots + 1 + ((i + 1) & 1) : d.dots, d.H + i + (int64_t)j * d.ldh));
        } else {
            for (int i = 0; i <= j; i++) {
                TRY(bdot(ctx, 0, Vcol(ctx, i), ctx->d_z, d.dots, ist, IGS_K_BLOCK_DOT));  // h = v_i . w
                TIMED(IGS_K_UPDATE, 24.0 * n,
                      launch_mgs_axpy(n, Vcol(ctx, i), ctx->d_z, d.dots + 1, d.H + i + (int64_t)j * d.ldh, ist, st));
            }
            TRY(bdot(ctx, 0, ctx->d_z, nullptr, d.dots, ist, IGS_K_BLOCK_DOT));          // ||w||^2
        }
        TIMED(IGS_K_SMALL, 0.0, launch_small(d, SS_MGS_NORM, 1, j + 1, m, t0, st));
        TIMED(IGS_K_UPDATE, 16.0 * n,
              launch_update(n, 0, ctx->d_V, ctx->ldv, ctx->d_z, nullptr, nullptr, nullptr,
                            d.scal + SC_GAMMA, Vcol(ctx, j + 1), nullptr, ist, j + 1, st));
        ctx->n_iter++;
        if (!ctx->capturing && (j + 1) % poll_every == 0 && j + 1 < m) {
            if (!ev[0]) {
                CUDA_TRY(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
                CUDA_TRY(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
            }
            CUDA_TRY(cudaMemcpyAsync(h_status + ev_slot, ist + ST_STATUS, sizeof(int), cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaEventRecord(ev[ev_slot], st));
            if (ev_pending >= 0) {
                TRY(wait_for(ctx, ev[ev_pending], nullptr, "igs_solve: checkpoint"));
                if (h_status[ev_pending] != RUNNING) break;
            }
            ev_pending = ev_slot;
            ev_slot ^= 1;
        }
    }
    if (!ctx->capturing) TRY(wait_for(ctx, nullptr, st, "igs_solve: cycle"));
    if (ev[0]) { cudaEventDestroy(ev[0]); cudaEventDestroy(ev[1]); }
    return IGS_OK;
}

// Run one cycle: for small single-GPU problems replay a captured CUDA graph of the whole
// cycle (p is baked into every node; the first iteration index t0 lives in device memory),
// otherwise enqueue it directly with status polling.
static igs_status launch_cycle(igs_ctx* ctx, int m, int alg, int t0) {
    cudaStream_t st = ctx->stream;
    ctx->h_pinned[40] = (double)t0;
    CUDA_TRY(cudaMemcpyAsync(ctx->dev_state.scal + SC_T0, ctx->h_pinned + 40, sizeof(double),
                             cudaMemcpyHostToDevice, st));
    // (G > 1 too: the halo send/recv, ncclAllReduce and the exchange kernels are captured;
    //  every rank captures the same sequence, and a stop inside the cycle turns the remaining
    //  work into no-ops while the collectives still run on every rank)
    const bool use_graph = ctx->graphs_enabled && !ctx->timing && !ctx->vsolve && !use_pcycle(ctx, alg) &&
                           ctx->n_local <= ((int64_t)1 << 21) && m <= 512 &&
                           (alg != IGS_ALG_MGS || (int64_t)m * (m + 7) / 2 <= 50000);  // MGS: O(m^2) nodes
    if (!use_graph) return run_cycle(ctx, m, alg, t0);
    // capture and replay on a private stream (the caller's may be the legacy default stream,
    // which cannot be captured); joined to the caller's stream with events
    if (!ctx->gstream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_g0, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_g1, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(ctx->ev_g0, st));
    CUDA_TRY(cudaStreamWaitEvent(ctx->gstream, ctx->ev_g0, 0));
    const auto key = std::make_pair(m, alg);
    auto itg = ctx->graphs.find(key);
    if (itg == ctx->graphs.end()) {
        cudaGraph_t g = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal));
        ctx->capturing = true;
        ctx->stream = ctx->gstream;
        const int64_t it0 = ctx->n_iter, r0 = ctx->n_reduce, a0 = ctx->n_allreduce, h0 = ctx->n_halo;
        igs_status s1 = run_cycle(ctx, m, alg, t0);
        ctx->stream = st;
        ctx->capturing = false;
        const int64_t dr = ctx->n_reduce - r0, da = ctx->n_allreduce - a0, dh = ctx->n_halo - h0;
        ctx->n_iter = it0;
        ctx->n_reduce = r0;
        ctx->n_allreduce = a0;
        ctx->n_halo = h0;
        cudaError_t e = cudaStreamEndCapture(ctx->gstream, &g);
        if (s1 != IGS_OK) { if (g) cudaGraphDestroy(g); return s1; }
        CUDA_TRY(e);
        cudaGraphExec_t ex = nullptr;
        e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        CUDA_TRY(e);
        itg = ctx->graphs.emplace(key, igs_ctx::CycleGraph{ex, dr, da, dh}).first;
    }
    CUDA_TRY(cudaGraphLaunch(itg->second.exec, ctx->gstream));
    ctx->n_reduce += itg->second.reductions;
    ctx->n_allreduce += itg->second.allreduces;
    ctx->n_halo += itg->second.halos;
    CUDA_TRY(cudaEventRecord(ctx->ev_g1, ctx->gstream));
    CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_g1, 0));
    ctx->n_graph_launches++;
    ctx->n_iter += m;
    return IGS_OK;
}

extern "C" igs_status igs_solve(igs_ctx* ctx, igs_mem vec_mem, const double* b, const double* x0,
                                int k, int restart, double tol, int gs_iters, igs_result* res) {
    ARG_CHECK(gs_iters == 1 || gs_iters == 2, "igs_solve: gs_iters must be 1 or 2");
    return igs_solve_alg(ctx, vec_mem, b, x0, k, restart, tol, gs_iters, res);
}

extern "C" igs_status igs_solve_alg(igs_ctx* ctx, igs_mem vec_mem, const double* b, const double* x0,
                                    int k, int restart, double tol, int algorithm, igs_result* res) {
    const int gs_iters = algorithm;
    if (ctx && ctx->aborted) {
        set_error("igs_solve: the communicator was aborted after an earlier failure; destroy the context");
        return IGS_ERR_STATE;
    }
    ARG_CHECK(ctx && ctx->ok, "igs_solve: bad context");
    ARG_CHECK(!ctx->vgroup || ctx->vsolve,
              "igs_solve: virtual-rank contexts (igs_create_virtual) run igs_virtual_spmv / igs_virtual_solve");
    ARG_CHECK(res && res->x && b, "igs_solve: NULL b / res / res->x");
    ARG_CHECK(algorithm >= IGS_ALG_IGS1 && algorithm <= IGS_ALG_MGS, "igs_solve_alg: unknown algorithm");
    ARG_CHECK(k >= 1 && (int64_t)k < ctx->n_global - 1, "igs_solve: need 1 <= k < n_global - 1 (P:873)");
    ARG_CHECK(restart >= 0, "igs_solve: restart < 0");
    ARG_CHECK(tol >= 0.0 && std::isfinite(tol), "igs_solve: tol must be finite and >= 0");
    ARG_CHECK(vec_mem == IGS_MEM_HOST || vec_mem == IGS_MEM_DEVICE, "igs_solve: bad memory kind");
    ARG_CHECK(vec_mem == IGS_MEM_HOST || (((uintptr_t)b % 16) == 0 && ((uintptr_t)res->x % 16) == 0),
              "igs_solve: device b and x need 16-byte alignment");
    CUDA_TRY(cudaSetDevice(ctx->dev));
    const int m1 = (restart > 0 && restart < k) ? restart : k;
    const bool hostv = vec_mem == IGS_MEM_HOST;
    TRY(ensure_workspace(ctx, m1, k, hostv));
    Dev& d = ctx->dev_state;
    cudaStream_t st = ctx->stream;
    const int64_t n = ctx->n_local;
    ctx->recs.clear();

    // vectors in HBM
    const double* db;
    double* dx;
    if (hostv) {
        TIMED(IGS_K_CYCLE, 0.0, {
            CUDA_TRY(cudaMemcpyAsync(ctx->d_b, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
            if (x0) CUDA_TRY(cudaMemcpyAsync(ctx->d_x, x0, sizeof(double) * n, cudaMemcpyHostToDevice, st));
            else CUDA_TRY(cudaMemsetAsync(ctx->d_x, 0, sizeof(double) * n, st));
        });
        db = ctx->d_b;
        dx = ctx->d_x;
    } else {
        db = b;
        dx = res->x;
        if (x0 && x0 != dx) CUDA_TRY(cudaMemcpyAsync(dx, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        else if (!x0) CUDA_TRY(cudaMemsetAsync(dx, 0, sizeof(double) * n, st));
    }
    const int64_t ar0 = ctx->n_allreduce;
    unsigned red0 = 0;  // reductions executed on the device (block dots that ran to completion)
    CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned_int + 24, ctx->d_counter + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    TRY(wait_for(ctx, nullptr, st, "igs_solve"));
    std::memcpy(&red0, ctx->h_pinned_int + 24, sizeof(unsigned));

    // ||b|| (one reduction; also the non-finite check of b)
    double* dsc = d.scal;
    TRY(bdot(ctx, 0, db, nullptr, d.dots, nullptr, IGS_K_CYCLE));
    double nb2 = 0.0;
    TRY(fetch(ctx, d.dots, 1, &nb2, nullptr, 0, nullptr));
    if (!std::isfinite(nb2)) {
        set_error("igs_solve: non-finite right-hand side");
        return IGS_ERR_NONFINITE;
    }
    const double nb = std::sqrt(nb2);
    std::vector<double> hres(k + 1, std::nan(""));
    res->iters = 0;
    res->cycles = 0;
    res->loo_frob = std::nan("");
    res->h_cols = 0;
    res->basis_cols = 0;
    res->term = IGS_TERM_MAXITER;
    if (res->H) std::fill(res->H, res->H + (size_t)(m1 + 1) * m1, 0.0);
    if (nb == 0.0) {
        CUDA_TRY(cudaMemsetAsync(dx, 0, sizeof(double) * n, st));
        if (hostv) CUDA_TRY(cudaMemcpyAsync(res->x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        TRY(wait_for(ctx, nullptr, st, "igs_solve"));
        res->term = IGS_TERM_CONVERGED;
        res->true_relres = 0.0;
        if (res->res_hist) res->res_hist[0] = 0.0;
        return IGS_OK;
    }
    {
        double hs[SC_COUNT] = {0};
        hs[SC_NB] = nb;
        hs[SC_TOL] = tol;
        hs[SC_ONE] = 1.0;
        CUDA_TRY(cudaMemcpyAsync(dsc, hs, sizeof(hs), cudaMemcpyHostToDevice, st));
    }
    int total = 0, cycles = 0, last_basis = 0;
    bool breakdown = false, x_sent = false;
    double rn = 0.0;
    for (;;) {
        // r = b - A x into z (not V[:,0]: the final basis must survive for the LOO
        // diagnostic); ||r||  (true residual at cycle start)
        TRY(spmv(ctx, dx, ctx->d_z, db, true, nullptr, IGS_K_CYCLE));
        TRY(bdot(ctx, 0, ctx->d_z, nullptr, d.dots, nullptr, IGS_K_CYCLE));
        double rn2 = 0.0;
        TRY(fetch(ctx, d.dots, 1, &rn2, nullptr, 0, nullptr));
        if (!std::isfinite(rn2)) {
            set_error("igs_solve: non-finite residual");
            return IGS_ERR_NONFINITE;
        }
        rn = std::sqrt(rn2);
        if (total == 0) hres[0] = rn / nb;
        if (breakdown) { res->term = IGS_TERM_BREAKDOWN; break; }
        if (tol > 0.0 && rn <= tol * nb) { res->term = IGS_TERM_CONVERGED; break; }
        if (total >= k) { res->term = IGS_TERM_MAXITER; break; }
        if (rn == 0.0) { res->term = IGS_TERM_CONVERGED; break; }
        const int m = std::min(m1, k - total);
        TRY(launch_cycle(ctx, m, gs_iters, total));
        int istate[ST_COUNT];
        TRY(fetch(ctx, nullptr, 0, nullptr, d.istate, ST_COUNT, istate));
        if (ctx->d_xchg) {  // the exchange barrier gave up on a peer (xchg.cuh): fail, do not hang
            int xerr = 0;
            TRY(fetch(ctx, nullptr, 0, nullptr, ctx->d_xerr, 1, &xerr));
            if (xerr)
                return abort_comm(ctx, "igs_solve: fused exchange barrier timeout after " +
                                           std::to_string(ctx->timeout_s) + " s (a peer rank did not arrive)");
        }
        const int status = istate[ST_STATUS], p = istate[ST_PDONE];
        if (status == STOP_NONFINITE) {
            set_error("igs_solve: non-finite value during the Arnoldi iteration");
            return IGS_ERR_NONFINITE;
        }
        if (cycles == 0) {
            res->h_cols = p;
            if (res->H)
                CUDA_TRY(cudaMemcpyAsync(res->H, d.H, sizeof(double) * (size_t)(m1 + 1) * m1, cudaMemcpyDeviceToHost, st));
        }
        // y = argmin ||rho e1 - H y|| ; x += V_p y
        TIMED(IGS_K_CYCLE, 0.0, launch_small(d, SS_LSQ, gs_iters, 0, m, total, st));
        // host vectors, and this cycle is the last (it runs to k: the loop ends after the
        // residual below): x += V_p y in 8 row chunks, each chunk's D2H on a copy stream
        // behind its update, so the PCIe copy of x overlaps the rest of the update
        const bool last_host = hostv && !ctx->timing && ctx->nranks == 1 && total + p >= k &&
                               status != STOP_BREAKDOWN && n >= 8 * 4096;
        if (last_host) {
            if (!ctx->cstream) {
                CUDA_TRY(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
                for (cudaEvent_t& e : ctx->ev_xc) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            const int64_t ch = round_up((n + 7) / 8, 256);
            for (int c = 0; c < 8; c++) {
                const int64_t r0 = (int64_t)c * ch, r1 = std::min<int64_t>(n, r0 + ch);
                if (r1 <= r0) break;
                launch_xupdate(r1 - r0, ctx->d_V + r0, ctx->ldv, d.y, dx + r0, d.istate, m, st);
                CUDA_TRY(cudaEventRecord(ctx->ev_xc[c], st));
                CUDA_TRY(cudaStreamWaitEvent(ctx->cstream, ctx->ev_xc[c], 0));
                CUDA_TRY(cudaMemcpyAsync(res->x + r0, dx + r0, sizeof(double) * (r1 - r0), cudaMemcpyDeviceToHost,
                                         ctx->cstream));
            }
            CUDA_TRY(cudaGetLastError());
            x_sent = true;
        } else {
            TIMED(IGS_K_CYCLE, 8.0 * n * p + 16.0 * n,
                  launch_xupdate(n, ctx->d_V, ctx->ldv, d.y, dx, d.istate, m, st));
        }
        total += p;
        cycles++;
        last_basis = istate[ST_BASIS];
        if (status == STOP_BREAKDOWN) breakdown = true;
    }
    res->iters = total;
    res->cycles = cycles;
    res->basis_cols = last_basis;
    res->true_relres = rn / nb;
    if (total > 0) CUDA_TRY(cudaMemcpyAsync(hres.data() + 1, d.res_hist + 1, sizeof(double) * total, cudaMemcpyDeviceToHost, st));
    std::vector<double> hl(k + 1, std::nan(""));
    if (res->lnorm_hist && total > 0 && gs_iters != IGS_ALG_MGS)
        CUDA_TRY(cudaMemcpyAsync(hl.data(), d.lnorm, sizeof(double) * (total + 1), cudaMemcpyDeviceToHost, st));
    res->s_norm = std::nan("");
    res->sigma_min = std::nan("");
    res->lgram_frob = std::nan("");
    // LOO of the final basis, ||S||_2 and sigma_min: diagnostics from G = V^T V
    if ((res->want_loo || res->want_basis_diag) && last_basis > 0) {
        const int c = last_basis;
        const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(64, n / 4096));
        const size_t need = (size_t)splits * c * c + (size_t)c * c + 2;
        if (need > ctx->gram_cap) {
            cudaFree(ctx->d_gram);
            ctx->d_gram = nullptr;
            CUDA_TRY(cudaMalloc(&ctx->d_gram, need * sizeof(double)));
            ctx->gram_cap = need;
        }
        double* G = ctx->d_gram + (size_t)splits * c * c;
        TIMED(IGS_K_CYCLE, 8.0 * n * c, launch_gram(n, c, ctx->d_V, ctx->ldv, ctx->d_gram, splits, G, st));
        TRY(allreduce(ctx, G, (int64_t)c * c));
        TIMED(IGS_K_CYCLE, 0.0, launch_loo_norm(c, G, G + (size_t)c * c, st));
        double loo[2] = {0.0, 0.0};
        TRY(fetch(ctx, G + (size_t)c * c, 2, loo, nullptr, 0, nullptr));
        if (res->want_loo) res->loo_frob = loo[0];
        res->lgram_frob = loo[1];
        if (res->want_basis_diag && c <= IGS_BASIS_DIAG_MAX) {  // larger bases: NaN (one-CTA Jacobi)
            double* ws = nullptr;
            CUDA_TRY(cudaMalloc(&ws, sizeof(double) * (basis_diag_doubles(c) + 2)));
            TIMED(IGS_K_CYCLE, 0.0, launch_basis_diag(c, G, ws, ws + basis_diag_doubles(c), st));
            double sd[2] = {0.0, 0.0};
            igs_status fs = fetch(ctx, ws + basis_diag_doubles(c), 2, sd, nullptr, 0, nullptr);
            cudaFree(ws);
            TRY(fs);
            res->s_norm = sd[0];
            res->sigma_min = sd[1];
        }
    }
    if (hostv && !x_sent) CUDA_TRY(cudaMemcpyAsync(res->x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    TRY(wait_for(ctx, nullptr, st, "igs_solve"));
    if (x_sent) CUDA_TRY(cudaStreamSynchronize(ctx->cstream));
    CUDA_TRY(cudaGetLastError());
    if (res->res_hist) std::memcpy(res->res_hist, hres.data(), sizeof(double) * (total + 1));
    if (res->lnorm_hist) {
        std::memcpy(res->lnorm_hist, hl.data(), sizeof(double) * (total + 1));
        if (total == 0 || gs_iters == IGS_ALG_MGS) res->lnorm_hist[0] = std::nan("");
    }
    if (res->H && res->h_cols < m1)  // columns past the last completed one are unspecified on
        std::fill(res->H + (size_t)(m1 + 1) * res->h_cols, res->H + (size_t)(m1 + 1) * m1, 0.0);
    res->allreduces = ctx->n_allreduce - ar0;
    {
        unsigned red1 = 0;
        CUDA_TRY(cudaMemcpyAsync(ctx->h_pinned_int + 24, ctx->d_counter + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        TRY(wait_for(ctx, nullptr, st, "igs_solve"));
        std::memcpy(&red1, ctx->h_pinned_int + 24, sizeof(unsigned));
        res->reductions = (int64_t)(red1 - red0);
    }
    TRY(timer_flush(ctx));
    return IGS_OK;
}

// ------------------------------------------------------------ virtual ranks (test hook)
extern "C" igs_status igs_create_virtual(igs_ctx** out, int nranks, int64_t n_global, const int64_t* bounds,
                                         const int64_t* rowptr, const void* colind, int colind_bits,
                                         const double* values, int cuda_device, void* cuda_stream) {
    ARG_CHECK(out && nranks >= 1 && n_global > 0 && bounds && rowptr && (colind_bits == 32 || colind_bits == 64),
              "igs_create_virtual: bad argument");
    ARG_CHECK(bounds[0] == 0 && bounds[nranks] == n_global, "igs_create_virtual: bounds must span [0, n_global)");
    for (int r = 0; r < nranks; r++) {
        out[r] = nullptr;
        ARG_CHECK(bounds[r + 1] >= bounds[r], "igs_create_virtual: bounds not monotone");
    }
    const size_t cb = colind_bits / 8;
    VirtPlan vp;
    vp.bounds.assign(bounds, bounds + nranks + 1);
    vp.ghosts.resize(nranks);
    std::vector<std::vector<int64_t>> rp(nranks);
    for (int r = 0; r < nranks; r++) {  // rank r's CSR block with local row offsets
        const int64_t r0 = bounds[r], nl = bounds[r + 1] - r0;
        rp[r].resize(nl + 1);
        for (int64_t i = 0; i <= nl; i++) rp[r][i] = rowptr[r0 + i] - rowptr[r0];
        const char* cr = static_cast<const char*>(colind) + cb * rowptr[r0];
        int64_t ng = 0;
        std::vector<int64_t> oc(nranks);
        TRY(igs_plan_ghosts(r0, nl, rp[r].data(), cr, colind_bits, nranks, bounds, &ng, nullptr, oc.data()));
        vp.ghosts[r].resize(ng);
        TRY(igs_plan_ghosts(r0, nl, rp[r].data(), cr, colind_bits, nranks, bounds, &ng, vp.ghosts[r].data(), oc.data()));
    }
    VGroup* g = new VGroup();
    g->G = nranks;
    g->members.assign(nranks, nullptr);
    for (int r = 0; r < nranks; r++) {
        const int64_t r0 = bounds[r], nl = bounds[r + 1] - r0;
        const char* cr = static_cast<const char*>(colind) + cb * rowptr[r0];
        igs_status st = create_ctx(&out[r], n_global, r0, nl, rp[r].data(), cr, colind_bits, values + rowptr[r0],
                                   rp[r][nl], IGS_MEM_HOST, cuda_device, nullptr, r, nranks, cuda_stream, &vp);
        if (st != IGS_OK) {
            const std::string msg = igs_last_error();
            for (int q = 0; q < r; q++) { out[q]->vgroup = nullptr; free_ctx(out[q]); out[q] = nullptr; }
            delete g;
            set_error(msg);
            return st;
        }
        out[r]->vgroup = g;
        g->members[r] = out[r];
        g->alive++;
    }
    return IGS_OK;
}

extern "C" igs_status igs_virtual_spmv(igs_ctx* const* ctxs, int nranks, const double* const* x, double* const* y,
                                       const double* const* b) {
    ARG_CHECK(ctxs && x && y && nranks >= 1, "igs_virtual_spmv: bad argument");
    VGroup* g = ctxs[0] ? ctxs[0]->vgroup : nullptr;
    ARG_CHECK(g && g->G == nranks, "igs_virtual_spmv: not one complete virtual group");
    for (int r = 0; r < nranks; r++)
        ARG_CHECK(ctxs[r] == g->members[r] && ((x[r] && y[r]) || ctxs[r]->n_local == 0),
                  "igs_virtual_spmv: contexts not in rank order / NULL vector");
    igs_ctx* c0 = ctxs[0];
    CUDA_TRY(cudaSetDevice(c0->dev));
    for (int r = 0; r < nranks; r++)  // every rank's send buffer first (the copies read them)
        launch_pack(ctxs[r]->n_send, ctxs[r]->d_send_idx, x[r], ctxs[r]->d_send, nullptr, ctxs[r]->stream);
    CUDA_TRY(cudaGetLastError());
    for (int r = 0; r < nranks; r++)
        TRY(spmv(ctxs[r], x[r], y[r], b ? b[r] : nullptr, b != nullptr, nullptr, IGS_K_SPMV));
    for (int r = 0; r < nranks; r++) TRY(wait_for(ctxs[r], nullptr, ctxs[r]->stream, "igs_virtual_spmv"));
    return IGS_OK;
}

extern "C" igs_status igs_virtual_solve(igs_ctx* const* ctxs, int nranks, const double* const* b, int k,
                                        int restart, double tol, int algorithm, igs_result* res) {
    ARG_CHECK(ctxs && b && res && nranks >= 1, "igs_virtual_solve: bad argument");
    VGroup* g = ctxs[0] ? ctxs[0]->vgroup : nullptr;
    ARG_CHECK(g && g->G == nranks, "igs_virtual_solve: not one complete virtual group");
    for (int r = 0; r < nranks; r++)
        ARG_CHECK(ctxs[r] == g->members[r] && (b[r] || ctxs[r]->n_local == 0) && (res[r].x || ctxs[r]->n_local == 0),
                  "igs_virtual_solve: contexts not in rank order / NULL vector");
    ARG_CHECK(k >= 1 && restart >= 0, "igs_virtual_solve: bad k / restart");
    CUDA_TRY(cudaSetDevice(ctxs[0]->dev));
    const int G = nranks;
    const int m1 = (restart > 0 && restart < k) ? restart : k;
    const size_t cap = std::max<size_t>((size_t)(m1 + 2) * (m1 + 2), 2 * (size_t)(m1 + 1) + 2);
    // events and staging (the members' threads only enqueue; nothing here is shared mutably)
    for (int q = 0; q < 2; q++)
        while ((int)g->ev_copy[q].size() < G) {
            cudaEvent_t a, c;
            CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
            g->ev_copy[q].push_back(a);
            g->ev_sum[q].push_back(c);
        }
    while ((int)g->ev_pack.size() < G) {
        cudaEvent_t a, c;
        CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
        g->ev_pack.push_back(a);
        g->ev_hcopy.push_back(c);
    }
    if (!g->d_stage_ptrs) CUDA_TRY(cudaMalloc(&g->d_stage_ptrs, sizeof(double*) * 2 * G));
    std::vector<const double*> hp(2 * (size_t)G);
    std::vector<cudaStream_t> saved(G), own(G, nullptr);
    for (int r = 0; r < G; r++) {
        igs_ctx* c = ctxs[r];
        if (c->vstage_cap < cap) {
            cudaFree(c->d_vstage);
            c->d_vstage = nullptr;
            CUDA_TRY(cudaMalloc(&c->d_vstage, sizeof(double) * 2 * cap));
            c->vstage_cap = cap;
        }
        hp[r] = c->d_vstage;
        hp[(size_t)G + r] = c->d_vstage + c->vstage_cap;
        c->v_ar_calls = c->v_halo_calls = 0;
    }
    CUDA_TRY(cudaMemcpy(g->d_stage_ptrs, hp.data(), sizeof(double*) * 2 * G, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaDeviceSynchronize());
    for (int r = 0; r < G; r++) {  // every member on its own stream and host thread
        saved[r] = ctxs[r]->stream;
        CUDA_TRY(cudaStreamCreateWithFlags(&own[r], cudaStreamNonBlocking));
        ctxs[r]->stream = own[r];
        ctxs[r]->vsolve = true;
    }
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->broken = false;
        g->arrived = 0;
        g->timeout_s = ctxs[0]->timeout_s;
    }
    std::vector<igs_status> st(G, IGS_OK);
    std::vector<std::string> msg(G);
    std::vector<std::thread> th;
    for (int r = 0; r < G; r++)
        th.emplace_back([&, r] {
            cudaSetDevice(ctxs[r]->dev);
            st[r] = igs_solve_alg(ctxs[r], IGS_MEM_DEVICE, b[r], nullptr, k, restart, tol, algorithm, &res[r]);
            if (st[r] != IGS_OK) {
                msg[r] = igs_last_error();
                g->fail();
            }
        });
    for (auto& t : th) t.join();
    cudaDeviceSynchronize();
    for (int r = 0; r < G; r++) {
        ctxs[r]->stream = saved[r];
        ctxs[r]->vsolve = false;
        cudaStreamDestroy(own[r]);
    }
    for (int r = 0; r < G; r++)
        if (st[r] != IGS_OK && msg[r].find("a member failed") == std::string::npos) {
            set_error("igs_virtual_solve: member " + std::to_string(r) + ": " + msg[r]);
            return st[r];
        }
    for (int r = 0; r < G; r++)
        if (st[r] != IGS_OK) {
            set_error("igs_virtual_solve: member " + std::to_string(r) + ": " + msg[r]);
            return st[r];
        }
    return IGS_OK;
}

extern "C" igs_status igs_stats(const igs_ctx* ctx, int64_t* allreduces, int64_t* halo_msgs,
                                int64_t* iterations) {
    ARG_CHECK(ctx != nullptr, "igs_stats: NULL context");
    if (allreduces) *allreduces = ctx->n_allreduce;
    if (halo_msgs) *halo_msgs = ctx->n_halo;
    if (iterations) *iterations = ctx->n_iter;
    return IGS_OK;
}

extern "C" igs_status igs_info(const igs_ctx* ctx, int key, int64_t* value) {
    ARG_CHECK(ctx != nullptr && value != nullptr, "igs_info: NULL argument");
    switch (key) {
        case IGS_INFO_XCHG: *value = ctx->d_xchg != nullptr; break;
        case IGS_INFO_NRANKS: *value = ctx->nranks; break;
        case IGS_INFO_NGHOST: *value = ctx->n_ghost; break;
        case IGS_INFO_NSEND: *value = ctx->n_send; break;
        case IGS_INFO_NPEERS: *value = (int64_t)ctx->peers.size(); break;
        case IGS_INFO_NBND: *value = ctx->A.n_bnd; break;
        case IGS_INFO_GRAPH_LAUNCHES: *value = ctx->n_graph_launches; break;
        case IGS_INFO_PCYCLE_LAUNCHES: *value = ctx->n_pcycle; break;
        case IGS_INFO_SELL: *value = ctx->A.sell_ptr != nullptr; break;
        case IGS_INFO_CSR_COMPACT: *value = ctx->csr_compact; break;
        case IGS_INFO_SELL_DIAG_SLICES: *value = ctx->sell_diag_slices; break;
        case IGS_INFO_PCYCLE_ARES: *value = ctx->last_ares; break;
        case IGS_INFO_SPMV_BYTES:
            *value = ctx->A.sell_ptr ? ctx->sell_stream_bytes + 8 * ctx->n_ghost : (int64_t)spmv_bytes(ctx);
            break;
        case IGS_INFO_SELL_WALK:
            *value = ctx->A.sell_ptr && ctx->A.sell_kind == 1 && ctx->A.sell_walk_min_n >= 0 &&
                     ctx->A.nrows >= ctx->A.sell_walk_min_n;
            break;
        default: ARG_CHECK(false, "igs_info: unknown key");
    }
    return IGS_OK;
}

extern "C" igs_status igs_set_timeout(igs_ctx* ctx, double seconds) {
    ARG_CHECK(ctx != nullptr && seconds > 0.0 && std::isfinite(seconds), "igs_set_timeout: bad argument");
    ctx->timeout_s = seconds;
    if (ctx->d_xchg && !ctx->aborted) {
        CUDA_TRY(cudaSetDevice(ctx->dev));
        ctx->h_xchg.timeout_ns = (unsigned long long)(seconds * 1e9);
        CUDA_TRY(cudaMemcpyAsync(ctx->d_xchg, &ctx->h_xchg, sizeof(XchgDev), cudaMemcpyHostToDevice, ctx->stream));
        TRY(wait_for(ctx, nullptr, ctx->stream, "igs_set_timeout"));
    }
    return IGS_OK;
}

extern "C" igs_status igs_set_timing(igs_ctx* ctx, int on) {
    ARG_CHECK(ctx != nullptr, "igs_set_timing: NULL context");
    ctx->timing = on != 0;
    if (on == 2) {
        for (int i = 0; i < IGS_K_COUNT; i++) { ctx->t_ms[i] = 0; ctx->t_bytes[i] = 0; ctx->t_launch[i] = 0; }
        ctx->tail_launches = 0;
    }
    return IGS_OK;
}

extern "C" igs_status igs_kernel_stats(const igs_ctx* ctx, int kind, double* ms, int64_t* launches,
                                       double* bytes) {
    ARG_CHECK(ctx != nullptr && kind >= 0 && kind < IGS_K_COUNT, "igs_kernel_stats: bad argument");
    if (ms) *ms = ctx->t_ms[kind];
    if (launches) *launches = ctx->t_launch[kind] + (kind == IGS_K_SMALL ? ctx->tail_launches : 0);
    if (bytes) *bytes = ctx->t_bytes[kind];
    return IGS_OK;
}

// ----------------------------------------------------------------- kernel entry points
static igs_status have_device() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error("no CUDA device (libigs has no CPU fallback)");
        return IGS_ERR_CUDA;
    }
    return IGS_OK;
}

extern "C" igs_status igs_op_block_dot(int64_t n, int p, const double* V, int64_t ld, const double* u,
                                       const double* z, double* out, void* cuda_stream) {
    ARG_CHECK(n >= 0 && p >= 0 && u && out && (p == 0 || V), "igs_op_block_dot: bad argument");
    ARG_CHECK(p == 0 || (ld >= n && ld % 2 == 0 && ((uintptr_t)V % 16) == 0), "igs_op_block_dot: V needs even ld >= n and 16-byte alignment");
    ARG_CHECK(((uintptr_t)u % 16) == 0 && (!z || ((uintptr_t)z % 16) == 0), "igs_op_block_dot: u, z need 16-byte alignment");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = bdot_grid_size(n, sms);
    double* part = nullptr;
    unsigned* counter = nullptr;
    CUDA_TRY(cudaMalloc(&part, sizeof(double) * (size_t)grid * 2 * (p + 1)));
    CUDA_TRY(cudaMalloc(&counter, 4 * sizeof(unsigned)));
    CUDA_TRY(cudaMemsetAsync(counter, 0, 4 * sizeof(unsigned), st));
    launch_block_dot(n, p, V, ld, u, z, out, part, counter, grid, nullptr, st);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(part);
    cudaFree(counter);
    CUDA_TRY(e);
    return IGS_OK;
}

// Measurement hook: `reps` back-to-back block dots (the solver's launch path) timed with
// CUDA events on cuda_stream; scratch allocated outside the timed region.
extern "C" igs_status igs_bench_block_dot(int64_t n, int p, const double* V, int64_t ld, const double* u,
                                          const double* z, double* out, int reps, float* ms,
                                          void* cuda_stream) {
    ARG_CHECK(n >= 1 && p >= 0 && u && out && ms && reps >= 1 && (p == 0 || V), "igs_bench_block_dot: bad argument");
    ARG_CHECK(p == 0 || (ld >= n && ld % 2 == 0 && ((uintptr_t)V % 16) == 0), "igs_bench_block_dot: V needs even ld >= n and 16-byte alignment");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = bdot_grid_size(n, sms);
    double* part = nullptr;
    unsigned* counter = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CUDA_TRY(cudaMalloc(&part, sizeof(double) * (size_t)grid * 2 * (p + 1)));
    CUDA_TRY(cudaMalloc(&counter, 4 * sizeof(unsigned)));
    struct Free { double* p; unsigned* c; cudaEvent_t a, b;
                  ~Free() { cudaFree(p); cudaFree(c); if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); } }
        guard{part, counter, nullptr, nullptr};
    CUDA_TRY(cudaEventCreate(&e0));
    guard.a = e0;
    CUDA_TRY(cudaEventCreate(&e1));
    guard.b = e1;
    CUDA_TRY(cudaMemsetAsync(counter, 0, 4 * sizeof(unsigned), st));
    launch_block_dot(n, p, V, ld, u, z, out, part, counter, grid, nullptr, st);  // warm-up
    CUDA_TRY(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; r++) launch_block_dot(n, p, V, ld, u, z, out, part, counter, grid, nullptr, st);
    CUDA_TRY(cudaEventRecord(e1, st));
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventSynchronize(e1));
    CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
    *ms /= (float)reps;
    return IGS_OK;
}

// Measurement hook: `reps` back-to-back fused updates (Alg. 3 form when alpha != NULL).
extern "C" igs_status igs_bench_update(int64_t n, int p, const double* V, int64_t ld, const double* u,
                                       const double* z, const double* alpha, const double* beta, double gamma,
                                       double* v_out, double* u_next, int reps, float* ms, void* cuda_stream) {
    ARG_CHECK(n >= 1 && p >= 0 && u && v_out && ms && reps >= 1 && (p == 0 || V), "igs_bench_update: bad argument");
    ARG_CHECK(!u_next || (z && beta), "igs_bench_update: u_next needs z and beta");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    double* dg = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CUDA_TRY(cudaMalloc(&dg, sizeof(double)));
    struct Free { double* g; cudaEvent_t a, b;
                  ~Free() { cudaFree(g); if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); } } guard{dg, nullptr, nullptr};
    CUDA_TRY(cudaEventCreate(&e0));
    guard.a = e0;
    CUDA_TRY(cudaEventCreate(&e1));
    guard.b = e1;
    CUDA_TRY(cudaMemcpyAsync(dg, &gamma, sizeof(double), cudaMemcpyHostToDevice, st));
    launch_update(n, p, V, ld, u, z, alpha, beta, dg, v_out, u_next, nullptr, 0, st);
    CUDA_TRY(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; r++) launch_update(n, p, V, ld, u, z, alpha, beta, dg, v_out, u_next, nullptr, 0, st);
    CUDA_TRY(cudaEventRecord(e1, st));
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventSynchronize(e1));
    CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
    *ms /= (float)reps;
    return IGS_OK;
}

// Algorithm 1: Q R = A with one or two Gauss-Seidel sweeps, on the solver's own
// kernels (block dot, small step, fused update).  Reductions per column: 1 (+1 for sweeps=2).
extern "C" igs_status igs_qr(int64_t n, int m, const double* A, int64_t lda, double* Q, int64_t ldq,
                             double* R, int sweeps, int64_t* reductions, void* cuda_stream) {
    ARG_CHECK(n >= 1 && m >= 1 && m <= n && A && Q && R && (sweeps == 1 || sweeps == 2), "igs_qr: bad argument");
    ARG_CHECK(lda >= n && ldq >= n && lda % 2 == 0 && ldq % 2 == 0 && ((uintptr_t)A % 16) == 0 &&
              ((uintptr_t)Q % 16) == 0, "igs_qr: A and Q need even leading dimensions >= n and 16-byte alignment");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = bdot_grid_size(n, sms);
    const size_t nsd = (size_t)m * m + 2 * (m + 1) + (m + 1) + 2 * (m + 1) + 2 + (size_t)grid * 2 * (m + 1);
    double* ws = nullptr;
    unsigned* counter = nullptr;
    CUDA_TRY(cudaMalloc(&ws, nsd * sizeof(double)));
    CUDA_TRY(cudaMalloc(&counter, 4 * sizeof(unsigned)));
    struct Free { double* w; unsigned* c; ~Free() { cudaFree(w); cudaFree(c); } } guard{ws, counter};
    CUDA_TRY(cudaMemsetAsync(ws, 0, nsd * sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(counter, 0, 4 * sizeof(unsigned), st));
    CUDA_TRY(cudaMemsetAsync(R, 0, sizeof(double) * (size_t)m * m, st));
    QrDev q;
    double* w = ws;
    q.R = R;
    q.L = w; w += (size_t)m * m;
    q.dots = w; w += 2 * (m + 1);
    q.dots2 = w; w += m + 1;
    q.alpha = w; w += m + 1;
    q.beta = w; w += m + 1;
    q.scal = w; w += 2;
    double* part = w;
    auto col = [&](const double* base, int64_t ld, int j) { return base + (int64_t)j * ld; };
    auto qcol = [&](int j) { return Q + (int64_t)j * ldq; };
    int64_t nred = 0;
    auto dot = [&](int p, const double* u, const double* z, double* out) {
        launch_block_dot(n, p, Q, ldq, u, z, out, part, counter, grid, nullptr, st);
        nred++;
    };
    // Step 1: R_11 = ||a_1||, q_1 = a_1 / R_11
    dot(0, col(A, lda, 0), nullptr, q.dots);
    launch_qr_small(q, QR_S0, 0, m, st);
    launch_update(n, 0, Q, ldq, col(A, lda, 0), nullptr, nullptr, nullptr, q.scal, qcol(0), nullptr,
                  nullptr, 0, st);
    if (m > 1) {
        // Step 2: R_12 = q_1^T a_2, w_2 = a_2 - R_12 q_1
        dot(0, qcol(0), col(A, lda, 1), q.dots);
        launch_qr_small(q, QR_S1, 1, m, st);
        launch_update(n, 0, Q, ldq, qcol(0), col(A, lda, 1), nullptr, q.beta, q.scal + 1,
                      qcol(0), qcol(1), nullptr, 0, st, q.scal + 1);
    }
    for (int k = 2; k <= m; k++) {
        const bool drain = (k == m);
        // Steps 4-5: ONE reduction [Q_{k-2}, w_{k-1}]^T [w_{k-1}, a_k]
        dot(k - 1, qcol(k - 1), drain ? nullptr : col(A, lda, k), q.dots);
        launch_qr_small(q, QR_CRIT, k, m, st);
        if (drain) {  // Step 6 for the last column
            launch_update(n, 0, Q, ldq, qcol(k - 1), nullptr, nullptr, nullptr, q.scal,
                          qcol(k - 1), nullptr, nullptr, 0, st);
            break;
        }
        // Steps 6, 10: q_{k-1} = w_{k-1} / gamma ; u_k = a_k - Q_{k-1} r1
        launch_update(n, k - 1, Q, ldq, qcol(k - 1), col(A, lda, k), nullptr, q.beta, q.scal,
                      qcol(k - 1), qcol(k), nullptr, 0, st, q.scal + 1);
        if (sweeps == 2) {
            // Steps 11-13: r2 = Q_{k-1}^T u_k (second reduction), r3 = (I+L)^{-1} r2, w_k = u_k - Q r3
            dot(k, qcol(k), nullptr, q.dots2);
            launch_qr_small(q, QR_CRIT2, k, m, st);
            launch_update(n, k, Q, ldq, qcol(k), nullptr, q.alpha, nullptr, q.scal + 1, qcol(k),
                          nullptr, nullptr, 0, st);
        }
    }
    CUDA_TRY(cudaGetLastError());
    std::vector<double> diag((size_t)m * m);
    CUDA_TRY(cudaMemcpyAsync(diag.data(), R, sizeof(double) * (size_t)m * m, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (reductions) *reductions = nred;
    for (int i = 0; i < m; i++) {
        const double d = diag[i + (size_t)i * m];
        if (!std::isfinite(d) || !(d > 0.0)) {
            set_error("igs_qr: column " + std::to_string(i) + " is (numerically) dependent or non-finite");
            return IGS_ERR_NONFINITE;
        }
    }
    return IGS_OK;
}

extern "C" igs_status igs_op_basis_diag(int64_t n, int c, const double* V, int64_t ld, double* out3,
                                        void* cuda_stream) {
    ARG_CHECK(n >= 1 && c >= 1 && c <= IGS_BASIS_DIAG_MAX && ld >= n && V && out3, "igs_op_basis_diag: bad argument");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(64, n / 4096));
    const size_t nd = (size_t)splits * c * c + (size_t)c * c + 2 + basis_diag_doubles(c) + 2;
    double* ws = nullptr;
    CUDA_TRY(cudaMalloc(&ws, nd * sizeof(double)));
    struct Free { double* w; ~Free() { cudaFree(w); } } guard{ws};
    double* G = ws + (size_t)splits * c * c;
    double* loo = G + (size_t)c * c;  // [||I - G||_F, ||tril(G, -1)||_F]
    double* dws = loo + 2;
    double* sd = dws + basis_diag_doubles(c);
    launch_gram(n, c, V, ld, ws, splits, G, st);
    launch_loo_norm(c, G, loo, st);
    launch_basis_diag(c, G, dws, sd, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out3, loo, sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(out3 + 1, sd, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return IGS_OK;
}

extern "C" igs_status igs_op_spmv(igs_ctx* ctx, const double* x, double* y) {
    ARG_CHECK(ctx && ctx->ok && x && y, "igs_op_spmv: bad argument");
    ARG_CHECK(ctx->nranks == 1, "igs_op_spmv: single-rank contexts only");
    CUDA_TRY(cudaSetDevice(ctx->dev));
    launch_spmv(ctx->A, x, y, nullptr, false, nullptr, ctx->stream);
    if (ctx->A.n_bnd > 0) launch_spmv_rows(ctx->A, x, y, nullptr, false, nullptr, ctx->stream);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return IGS_OK;
}

extern "C" igs_status igs_op_update(int64_t n, int p, const double* V, int64_t ld, const double* u,
                                    const double* z, const double* alpha, const double* beta,
                                    double gamma, double* v_out, double* u_next, void* cuda_stream) {
    ARG_CHECK(n >= 0 && p >= 0 && u && v_out && (p == 0 || V), "igs_op_update: bad argument");
    ARG_CHECK(!u_next || (z && beta), "igs_op_update: u_next needs z and beta");
    ARG_CHECK(p == 0 || (ld >= n && ld % 2 == 0 && ((uintptr_t)V % 16) == 0), "igs_op_update: V needs even ld >= n and 16-byte alignment");
    ARG_CHECK(((uintptr_t)u % 16) == 0 && (!z || ((uintptr_t)z % 16) == 0), "igs_op_update: u, z need 16-byte alignment");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    double* dg = nullptr;
    CUDA_TRY(cudaMalloc(&dg, sizeof(double)));
    CUDA_TRY(cudaMemcpyAsync(dg, &gamma, sizeof(double), cudaMemcpyHostToDevice, st));
    launch_update(n, p, V, ld, u, z, alpha, beta, dg, v_out, u_next, nullptr, 0, st);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dg);
    CUDA_TRY(e);
    return IGS_OK;
}

extern "C" igs_status igs_op_trisolve(int order, const double* L, int ldl, const double* b, double* x,
                                      void* cuda_stream) {
    ARG_CHECK(order >= 0 && ldl >= order && (order == 0 || (L && b && x)), "igs_op_trisolve: bad argument");
    TRY(have_device());
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    launch_trisolve(order, L, ldl, b, x, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(st));
    return IGS_OK;
}
