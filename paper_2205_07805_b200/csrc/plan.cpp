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
#include "sell_plan.h"

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

// ---------------------------------------------------------------- SELL-32 layout (sell_plan.h)
namespace igs {

void sell_plan(int64_t n, const int64_t* rowptr, const int64_t* local_col, const double* values,
               const std::vector<int64_t>& bnd, bool want_diag, SellHost& out) {
    constexpr int SELL_BOUNDARY = 255;
    const int64_t ns = (n + 31) / 32;
    std::vector<int64_t> sp((size_t)ns + 1, 0);
    std::vector<uint8_t> len((size_t)n);
    std::vector<int64_t> cp((size_t)ns + 1, 0);
    std::vector<int32_t> dg((size_t)ns * 8, 0);
    std::vector<uint8_t> mk((size_t)n, 0);
    int64_t ctot = 0, ndiag = 0;
    size_t bi = 0;
    for (int64_t s = 0; s < ns; s++) {
        const int64_t r0 = 32 * s, r1 = std::min<int64_t>(n, r0 + 32);
        int64_t mx = 0;
        for (int64_t r = r0; r < r1; r++) {
            if (bi < bnd.size() && bnd[bi] == r) { len[(size_t)r] = SELL_BOUNDARY; bi++; continue; }
            const int64_t l = rowptr[r + 1] - rowptr[r];
            if (l >= SELL_BOUNDARY) { out = SellHost(); return; }  // long rows: no SELL copy
            len[(size_t)r] = (uint8_t)l;
            mx = std::max(mx, l);
        }
        bool ok = want_diag;
        int64_t D[8];
        int nd = 0;
        for (int64_t r = r0; r < r1 && ok; r++) {
            if (len[(size_t)r] == SELL_BOUNDARY) continue;
            int64_t prev = INT64_MIN;
            for (int64_t q = rowptr[r]; q < rowptr[r + 1] && ok; q++) {
                const int64_t c = local_col[(size_t)q], o = c - r;
                if (c < 0 || c >= n || o <= prev || o > INT32_MAX || o < INT32_MIN) { ok = false; break; }
                prev = o;
                bool seen = false;
                for (int i = 0; i < nd; i++) seen = seen || D[i] == o;
                if (!seen) {
                    if (nd == 8) { ok = false; break; }
                    D[nd++] = o;
                }
            }
        }
        if (ok) {
            std::sort(D, D + nd);
            for (int i = 0; i < nd; i++) dg[(size_t)s * 8 + i] = (int32_t)D[i];
            for (int64_t r = r0; r < r1; r++) {
                if (len[(size_t)r] == SELL_BOUNDARY) continue;
                unsigned m = 0;
                for (int64_t q = rowptr[r]; q < rowptr[r + 1]; q++) {
                    const int64_t o = local_col[(size_t)q] - r;
                    m |= 1u << (int)(std::lower_bound(D, D + nd, o) - D);
                }
                mk[(size_t)r] = (uint8_t)m;
            }
            ndiag++;
            sp[(size_t)s + 1] = sp[(size_t)s] + 32 * nd;
        } else {
            sp[(size_t)s + 1] = sp[(size_t)s] + 32 * mx;
            ctot += 32 * mx;
        }
        cp[(size_t)s + 1] = ctot;
    }
    const int64_t tot = std::max<int64_t>(sp[(size_t)ns], 1);
    std::vector<double> sv((size_t)tot, 0.0);
    std::vector<int64_t> sc((size_t)std::max<int64_t>(ctot, 1), 0);
    for (int64_t r = 0; r < n; r++) {
        if (len[(size_t)r] == SELL_BOUNDARY) continue;
        const int64_t s = r >> 5, base = sp[(size_t)s] + (r & 31), cb = cp[(size_t)s] + (r & 31);
        const bool diag = cp[(size_t)s + 1] == cp[(size_t)s];
        const int32_t* D = dg.data() + 8 * s;
        const int nd = (int)((sp[(size_t)s + 1] - sp[(size_t)s]) / 32);
        for (int64_t q = rowptr[r], k = 0; q < rowptr[r + 1]; q++, k++) {
            if (diag) {
                const int jpos = (int)(std::lower_bound(D, D + nd, (int32_t)(local_col[(size_t)q] - r)) - D);
                sv[(size_t)(base + 32 * jpos)] = values[q];
                continue;
            }
            sv[(size_t)(base + 32 * k)] = values[q];
            const int64_t at = cb + 32 * k;
            sc[(size_t)at] = local_col[(size_t)q];
        }
    }
    // row lengths and masks padded to whole slices (the kernels read whole slices)
    len.resize((size_t)ns * 32, 0);
    mk.resize((size_t)ns * 32, 0);
    out.ptr.swap(sp);
    out.cptr.swap(cp);
    out.diag.swap(dg);
    out.len.swap(len);
    out.mask.swap(mk);
    out.val.swap(sv);
    out.col.swap(sc);
    out.ndiag = ndiag;
    out.built = true;
}

}  // namespace igs

extern "C" igs_status igs_plan_sell(int64_t n, const int64_t* rowptr, const int64_t* local_col,
                                    const double* values, int want_diag, int64_t n_bnd,
                                    const int64_t* bnd_rows, int64_t* ptr, int64_t* cptr, int32_t* diag,
                                    uint8_t* len, uint8_t* mask, int64_t cap_val, double* val,
                                    int64_t cap_col, int64_t* col, int64_t* n_val, int64_t* n_col,
                                    int64_t* n_diag) {
    if (n < 0 || !rowptr || (rowptr[n] > 0 && (!local_col || !values)) || n_bnd < 0 || (n_bnd > 0 && !bnd_rows) ||
        !n_val || !n_col || !n_diag) {
        igs::set_error("igs_plan_sell: bad argument");
        return IGS_ERR_ARG;
    }
    for (int64_t i = 0; i < n_bnd; i++)
        if (bnd_rows[i] < 0 || bnd_rows[i] >= n || (i > 0 && bnd_rows[i] <= bnd_rows[i - 1])) {
            igs::set_error("igs_plan_sell: bnd_rows must be ascending rows in [0, n)");
            return IGS_ERR_ARG;
        }
    igs::SellHost h;
    igs::sell_plan(n, rowptr, local_col, values, std::vector<int64_t>(bnd_rows, bnd_rows + n_bnd), want_diag != 0, h);
    if (!h.built) { *n_val = -1; *n_col = -1; *n_diag = 0; return IGS_OK; }
    const int64_t ns = (n + 31) / 32;
    *n_val = h.ptr[(size_t)ns];
    *n_col = h.cptr[(size_t)ns];
    *n_diag = h.ndiag;
    if (ptr) std::memcpy(ptr, h.ptr.data(), sizeof(int64_t) * (size_t)(ns + 1));
    if (cptr) std::memcpy(cptr, h.cptr.data(), sizeof(int64_t) * (size_t)(ns + 1));
    if (diag && ns) std::memcpy(diag, h.diag.data(), sizeof(int32_t) * (size_t)(8 * ns));
    if (len && ns) std::memcpy(len, h.len.data(), (size_t)(32 * ns));
    if (mask && ns) std::memcpy(mask, h.mask.data(), (size_t)(32 * ns));
    if (val) {
        if (cap_val < *n_val) { igs::set_error("igs_plan_sell: cap_val too small"); return IGS_ERR_ARG; }
        if (*n_val) std::memcpy(val, h.val.data(), sizeof(double) * (size_t)*n_val);
    }
    if (col) {
        if (cap_col < *n_col) { igs::set_error("igs_plan_sell: cap_col too small"); return IGS_ERR_ARG; }
        if (*n_col) std::memcpy(col, h.col.data(), sizeof(int64_t) * (size_t)*n_col);
    }
    return IGS_OK;
}
