// sell_plan.h -- host-only layout of the SELL-32 copy of a CSR row block (plan.cpp); used by
// igs_create (api.cu uploads the arrays) and by igs_plan_sell (CPU tests).  DESIGN.md §5, §6.
#pragma once
#include <cstdint>
#include <vector>

namespace igs {

struct SellHost {
    std::vector<int64_t> ptr;    // [ns + 1] value offset of slice s (multiples of 32)
    std::vector<int64_t> cptr;   // [ns + 1] column offset; cptr[s+1] == cptr[s]: diagonal slice
    std::vector<int32_t> diag;   // [8 ns]   offsets c - r of a diagonal slice, ascending
    std::vector<uint8_t> len;    // [32 ns]  nonzeros per row; 255 = boundary row (not stored)
    std::vector<uint8_t> mask;   // [32 ns]  list positions a row of a diagonal slice uses
    std::vector<double> val;     // [max(ptr[ns], 1)]
    std::vector<int64_t> col;    // [max(cptr[ns], 1)] local columns of the explicit slices
    int64_t ndiag = 0;           // diagonal slices
    bool built = false;          // false: some row has >= 255 entries (no SELL copy)
};

// Slices of 32 rows.  A slice whose rows (boundary rows aside) have every column in [0, n),
// offsets c - r strictly increasing along each row and at most 8 distinct offsets in the
// slice is *diagonal* (when want_diag): it lists its offsets in ascending order and stores
// the entry of row 32s+l with offset list[j] at ptr[s] + 32j + l (bit j of the row's mask
// set; rows without that offset keep a zero there).  Any other slice is *explicit*: entry k
// of row 32s+l (CSR order) at ptr[s] + 32k + l, its column at cptr[s] + 32k + l, padded to
// the slice's longest row.  bnd: ascending rows left out (len 255, mask 0, nothing stored).
void sell_plan(int64_t n, const int64_t* rowptr, const int64_t* local_col, const double* values,
               const std::vector<int64_t>& bnd, bool want_diag, SellHost& out);

}  // namespace igs
