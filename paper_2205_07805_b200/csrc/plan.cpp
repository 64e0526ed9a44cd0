// plan.cpp -- host-only row-block partition / halo planning for libigs (no device needed).
//
// Rank r owns rows [bounds[r], bounds[r+1]) of A, of every n-vector and of V.  Its CSR
// block references global columns; the ones outside its own range are "ghosts", received
// each iteration from their owners before the SpMV (row-block SpMV).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/igs.h"

namespace igs {
void set_error(const std::string& msg);
}

namespace {

inline int64_t colat(const void* colind, int bits, int64_t q) {
    return bits == 64 ? static_cast<const int64_t*>(colind)[q]
                      : static_cast<int64_t>(static_cast<const int32_t*>(colind)[q]);
}

}  // namespace

extern "C" igs_status igs_plan_ghosts(int64_t row_begin, int64_t n_local, const int64_t* rowptr,
                                      const void* colind, int colind_bits, int nranks,
                                      const int64_t* bounds, int64_t* n_ghost, int64_t* ghosts,
                                      int64_t* ghost_owner_count) {
    if (n_local < 0 || (n_local > 0 && (!rowptr || !colind)) || !n_ghost ||
        (colind_bits != 32 && colind_bits != 64) || nranks < 1 || !bounds) {
        igs::set_error("igs_plan_ghosts: invalid argument");
        return IGS_ERR_ARG;
    }
    const int64_t row_end = row_begin + n_local;
    std::vector<int64_t> g;
    const int64_t nnz = n_local > 0 ? rowptr[n_local] : 0;
    for (int64_t q = 0; q < nnz; q++) {
        const int64_t c = colat(colind, colind_bits, q);
        if (c < row_begin || c >= row_end) g.push_back(c);
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    if (ghosts && *n_ghost < (int64_t)g.size()) {
        igs::set_error("igs_plan_ghosts: ghosts capacity too small");
        return IGS_ERR_ARG;
    }
    *n_ghost = (int64_t)g.size();
    if (ghosts) std::memcpy(ghosts, g.data(), g.size() * sizeof(int64_t));
    if (ghost_owner_count) {
        for (int q = 0; q < nranks; q++) ghost_owner_count[q] = 0;
        int q = 0;
        for (int64_t c : g) {
            while (q < nranks && c >= bounds[q + 1]) q++;
            if (q >= nranks || c < bounds[q]) {
                igs::set_error("igs_plan_ghosts: column outside every rank's row block");
                return IGS_ERR_ARG;
            }
            ghost_owner_count[q]++;
        }
    }
    return IGS_OK;
}

extern "C" igs_status igs_plan_remap(int64_t row_begin, int64_t n_local, const int64_t* rowptr,
                                     const void* colind, int colind_bits, int64_t n_ghost,
                                     const int64_t* ghosts, int64_t* local_colind) {
    if (n_local < 0 || (n_local > 0 && (!rowptr || !colind || !local_colind)) ||
        (n_ghost > 0 && !ghosts) || (colind_bits != 32 && colind_bits != 64)) {
        igs::set_error("igs_plan_remap: invalid argument");
        return IGS_ERR_ARG;
    }
    const int64_t row_end = row_begin + n_local;
    const int64_t nnz = n_local > 0 ? rowptr[n_local] : 0;
    for (int64_t q = 0; q < nnz; q++) {
        const int64_t c = colat(colind, colind_bits, q);
        if (c >= row_begin && c < row_end) {
            local_colind[q] = c - row_begin;
        } else {
            const int64_t* it = std::lower_bound(ghosts, ghosts + n_ghost, c);
            if (it == ghosts + n_ghost || *it != c) {
                igs::set_error("igs_plan_remap: column missing from the ghost list");
                return IGS_ERR_ARG;
            }
            local_colind[q] = n_local + (it - ghosts);
        }
    }
    return IGS_OK;
}
