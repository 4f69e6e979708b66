// internal.h -- host-side helpers shared by the product's C++/CUDA sources.
// (Product side only; the oracle under oracle/ shares nothing with this.)
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dls_b200.h"

namespace dls {

// Section 2.3 plan of a problem.
struct Plan {
    int n = 0;
    bool vs = false;
    bool fixed_first_row = false;
    std::vector<int> cells;      // i*n+j in fill order
    std::vector<uint8_t> forced; // 1 = taken by the forced-cell rule
    int diag_depth = 0;          // first depth covering both diagonals
    int hourglass_depth = 0;     // hourglass plans: depth covering row N-1 too
    std::vector<uint8_t> pre;    // n*n, 1 = assigned a priori (not planned)
};

// Returns false on bad arguments.
bool make_plan(int n, bool vs, bool fixed_first_row, Plan *out);

// Section 2.3 order below an arbitrary a-priori pattern `pre` (n*n), taking the
// cells of `head` first (in that order) and then the V-score / forced rule.
bool make_plan_from(int n, bool vs, const uint8_t *pre, const std::vector<int> &head, Plan *out);

// Hourglass plan (Section 4.3): row 0 fixed, the diagonal cells in the
// standard order, then the cells of row N-1, then the rule of Section 2.3.
bool make_hourglass_plan(int n, bool vs, Plan *out);

// Validity of (n, symmetric) combinations.
bool valid_problem(int n, int symmetric, int fixed_first_row);

// Children of `n_in` depth-d0 records at depth d1 (plan cells [d0, d1)), with
// the index of their parent record.  Writes up to `capacity` records, returns the
// total.  extra_nodes (optional) = partial squares at depths d0+1 .. d1.
int64_t refine(const Plan &plan, int d0, int d1, const uint8_t *in, int64_t n_in, uint8_t *out,
               uint32_t *parent, int64_t capacity, int64_t *extra_nodes);

// Host-side check that a record is a consistent depth-`depth` prefix of `plan`.
bool valid_record(const Plan &plan, int depth, const uint8_t *rec);

// dls_count for an arbitrary plan (count.cu).
// Records are refined on the host (P:481 below each record) when fewer than
// refine_below (< 0: the default, ~1 per lane) are given.
// Scratch device memory from the library's own stream-ordered pool (one per
// device, freed memory kept cached up to 1 GB); free with cudaFreeAsync.
cudaError_t scratch_alloc(void **ptr, size_t bytes, cudaStream_t stream);
void scratch_trim(size_t keep_bytes);
int count_records(const Plan &plan, int depth, const uint8_t *prefix_buf, int64_t n_prefix, uint64_t *out_counts,
                  uint64_t *out_total, uint64_t *out_nodes, void *stream, int64_t refine_below = -1);

void set_error(const std::string &msg);
const char *get_error();

}  // namespace dls
