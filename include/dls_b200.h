/*
 * dls_b200.h -- C ABI of the B200 (sm_100a) diagonal-Latin-square enumerator.
 *
 * Implements the data-parallel hot path of Kochemazov, Vatutin, Zaikin, "Fast
 * Algorithm for Enumerating Diagonal Latin Squares of Small Order"
 * (arXiv:1709.02599).  "P:<n>" cites line n of the paper's PAPER.md.
 *
 * Terms
 *   order n        1 <= n <= 10 (the paper's range: "order at most 9 ... 10").
 *   symmetric      0 = diagonal Latin squares (DLS);
 *                  1 = vertically symmetric DLS, LS[i][j] = n-1-LS[i][n-1-j]
 *                      (P:520-522); even n only.
 *   fixed_first_row 1 = row 0 is assigned a priori to 0..n-1 (normalisation);
 *                  0 = row 0 is searched like every other row.
 *   plan           the cell order of Section 2.3: repeatedly take the
 *                  last free cell of any row/column/diagonal with n-1 assigned
 *                  cells (rows, then columns, then main diagonal, then antidiagonal),
 *                  else the free cell with the largest V = r_i + c_j + md + ad,
 *                  lexicographically first among ties.  For symmetric=1 only
 *                  left-half cells (j <= n-1-j) are planned; taking (i,j) also
 *                  assigns its mirror (i,n-1-j) (reading R4).
 *   prefix record  n*n bytes, row-major, cell value 0..n-1 or DLS_EMPTY (0xFF).
 *                  A depth-d prefix assigns exactly row 0 (if fixed_first_row),
 *                  the first d plan cells (and their mirrors when symmetric), and
 *                  nothing else: a workunit of P:481.
 *   diag depth     the smallest d whose prefixes assign every cell of the main
 *                  diagonal and antidiagonal.  dls_count needs depth >= diag depth
 *                  (the GPU search then only tracks row and column sets).
 *   count          number of complete (symmetric) DLS that extend a prefix.
 *   node           a consistent partial square visited below a prefix (each
 *                  successful cell assignment of the searched levels, see
 *                  dls_search_levels); the unit of "search nodes/sec".
 *
 * Error behaviour: every call returns a negative DLS_E_* code on failure and
 * writes nothing it did not document as written.  No call aborts the process.
 * Thread safety: calls are reentrant; dls_count serialises on its own stream.
 * Device memory: per-launch scratch (the 2 MB donation pool, the symmetry-breaking
 * buffers) comes from the library's own stream-ordered memory pool (one per
 * device, created on first use; freed scratch stays cached up to 1 GB,
 * DLS_POOL_KEEP=<bytes> in the environment changes that; dls_count_sb trims it
 * back to 64 MB on return).  The process's default pool is not touched.
 */
#ifndef DLS_B200_H
#define DLS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DLS_EMPTY 0xFF
#define DLS_MAX_ORDER 10

#define DLS_OK 0
#define DLS_E_ARG (-1)         /* bad order / depth / flag / null pointer        */
#define DLS_E_CUDA (-2)        /* a CUDA runtime call failed (see dls_last_error) */
#define DLS_E_PREFIX (-3)      /* a prefix record is not a consistent depth-d prefix */
#define DLS_E_NODEVICE (-4)    /* no CUDA device: the GPU path is the only path  */

/* Version string of the library ("dls_b200 <semver> sm_100a"). */
const char *dls_version(void);

/* Human-readable text of the last error on the calling thread ("" if none). */
const char *dls_last_error(void);

/*
 * dls_plan -- the Section 2.3 cell order (Fig. 1 for n = 9).
 *   out_cells      host, capacity n*n int32: cells as i*n+j in fill order
 *                  (row 0 excluded when fixed_first_row; left half only when
 *                  symmetric).
 *   out_forced     host, capacity n*n uint8 or NULL: 1 where the step was taken
 *                  by the forced-cell rule of P:154 / Section 2.4.1.
 *   out_n_steps    host: number of cells written.
 *   out_diag_depth host: diag depth (see Terms).
 * Returns DLS_OK or DLS_E_ARG.
 */
int dls_plan(int n, int symmetric, int fixed_first_row,
             int32_t *out_cells, uint8_t *out_forced,
             int32_t *out_n_steps, int32_t *out_diag_depth);

/*
 * dls_split -- the workunit decomposition of P:481: every consistent assignment
 * of the first `depth` plan cells (0 <= depth <= n_steps), in depth-first order
 * with candidate values increasing at every cell (rightmost-bit order of Alg. 4,
 * P:242-243).
 *   out_prefixes   host, capacity*n*n bytes (prefix records) or NULL.
 *   capacity       number of records out_prefixes can hold.
 * Writes min(total, capacity) records and returns total (int64, may exceed
 * capacity: call with NULL/0 first to size the buffer), or a DLS_E_* code.
 */
int64_t dls_split(int n, int symmetric, int fixed_first_row, int depth,
                  uint8_t *out_prefixes, int64_t capacity);

/*
 * dls_emit -- the optional compact emit of squares (small n): the same search as
 * dls_count_async, but every completed square is written as an n*n record
 * (row-major values) into d_out, in no particular order.
 *   d_prefixes     device, n_prefix depth-`depth` records;
 *   d_out          device, capacity*n*n bytes (capacity may be 0: count only).
 * Synchronous.  Returns the number of completions (records written: min(that,
 * capacity)), or a DLS_E_* code.
 */
int64_t dls_emit(int n, int symmetric, int fixed_first_row, int depth,
                 const uint8_t *d_prefixes, int64_t n_prefix,
                 uint8_t *d_out, int64_t capacity, void *stream);

/*
 * dls_refine -- the same decomposition applied below given records: every
 * consistent assignment of plan cells [depth, depth2) below each of the n_in
 * depth-`depth` records `in` (host), in record order then depth-first order.
 *   out            host, capacity*n*n bytes or NULL; parent: host, capacity
 *                  uint32 (index of the record each output extends) or NULL.
 * Returns the total number of output records (may exceed capacity), DLS_E_ARG, or
 * DLS_E_PREFIX if some input record is not a consistent depth-`depth` prefix.
 */
int64_t dls_refine(int n, int symmetric, int fixed_first_row, int depth,
                   const uint8_t *in, int64_t n_in, int depth2,
                   uint8_t *out, uint32_t *parent, int64_t capacity);

/*
 * dls_count -- exhaustive completion count of every prefix (Alg. 4, P:235-258,
 * run on the B200: one prefix per lane of a persistent sm_100a kernel, an
 * explicit per-lane stack, a global atomic work queue and warp-level subtree
 * donation).
 *   prefix_buf     n_prefix depth-`depth` prefix records; host or device memory
 *                  (detected; host buffers are staged to the device inside the call).
 *   out_counts     n_prefix uint64 completion counts (host or device) or NULL.
 *   out_total      host uint64: sum of all counts, or NULL.
 *   out_nodes      host uint64: search nodes visited, or NULL.
 *   stream         cudaStream_t to run on (NULL = legacy default stream).
 * Synchronous: returns after the results are written.  Returns DLS_OK,
 * DLS_E_ARG (depth < diag depth, bad sizes), DLS_E_PREFIX (some record is not a
 * consistent depth-`depth` prefix; its count is 0), DLS_E_CUDA, DLS_E_NODEVICE.
 */
int dls_count(int n, int symmetric, int fixed_first_row, int depth,
              const uint8_t *prefix_buf, int64_t n_prefix,
              uint64_t *out_counts, uint64_t *out_total, uint64_t *out_nodes,
              void *stream);

/*
 * dls_search_levels -- number of plan cells the GPU search assigns below a
 * depth-`depth` record: n_steps - depth, or fewer when the two-row closure applies
 * (DESIGN.md "Tail closure"): at the first level after which only two rows have
 * empty cells, in the same columns and off both diagonals, the search stops and
 * counts the completions in closed form (GF(2) rank of the columns' missing
 * pairs).  The nodes dls_count reports are the assignments of these levels
 * (R15).  The environment variable DLS_CLOSE=0 turns the closure off
 * (full search; diagnostics and A/B).
 *   out_levels     host int32.
 * Returns DLS_OK or DLS_E_ARG.
 */
int dls_search_levels(int n, int symmetric, int fixed_first_row, int depth, int32_t *out_levels);

/*
 * dls_count_async -- the same search, enqueued on `stream` without waiting.
 * All pointers are DEVICE memory:
 *   d_prefixes     n_prefix prefix records.
 *   d_counts       n_prefix uint64 or NULL (zeroed by the call).
 *   d_stats        DLS_STATS_WORDS uint64 (zeroed by the call); after the stream
 *                  completes: [0] total count, [1] search nodes (every cell
 *                  assignment below the records, complete squares included), [2] error word
 *                  (bit 0: some record was inconsistent; bits 8..: internal
 *                  invariants violated -- only the checked build
 *                  libdls_b200_checked.so, compiled with -DDLS_CHECKS, sets
 *                  them; dls_count then returns DLS_E_CUDA), [3] work-queue
 *                  cursor, [4] subtree donations, [5] busy lane-bursts,
 *                  [6] lane-bursts (lane utilisation = [5]/[6]), [7] subtrees
 *                  published to the device-wide donation pool, [8] two-row
 *                  states counted in closed form (dls_search_levels), [9] 0.
 * Returns DLS_OK or DLS_E_ARG/DLS_E_CUDA/DLS_E_NODEVICE for launch-time errors.
 */
#define DLS_STATS_WORDS 10
int dls_count_async(int n, int symmetric, int fixed_first_row, int depth,
                    const uint8_t *d_prefixes, int64_t n_prefix,
                    uint64_t *d_counts, uint64_t *d_stats, void *stream);

/*
 * dls_canonize -- Alg. 5 on the GPU for hourglass designs (row 0 =
 * 0..n-1, both diagonals and row n-1 assigned): out_mult[i] = 0 if record
 * i is not the lexicographically smallest design of its class under the
 * M-transformations that keep hourglass designs, else the number of
 * designs in its class.  The group: symmetric pairs of rows+columns permuted with
 * pair {0, n-1} in place, each pair optionally swapped, columns optionally
 * mirrored (the mirror is left out when symmetric: P:524).  3 <= n <= 10.
 *   hourglasses    n_rec records (host or device); out_mult n_rec uint32 (host or device).
 */
int dls_canonize(int n, int symmetric, const uint8_t *hourglasses, int64_t n_rec,
                 uint32_t *out_mult, void *stream);

/*
 * dls_count_sb -- the symmetry-broken enumeration of Alg. 6 for the
 * first-row-fixed problem: every hourglass design is generated and canonised on
 * the GPU, the completions of each canonic design are counted by the search
 * kernel (plan: diagonals, row n-1, then Section 2.3) and multiplied by its class
 * size (Corollary 1).
 *   out_total       host: number of (vertically symmetric) DLS, first row fixed;
 *   out_hourglasses host: hourglass designs generated; out_classes: canonic ones;
 *   out_nodes       host: search nodes below the canonic designs.
 * Synchronous.  3 <= n <= 10 (even when symmetric).
 */
int dls_count_sb(int n, int symmetric, uint64_t *out_total, uint64_t *out_hourglasses,
                 uint64_t *out_classes, uint64_t *out_nodes, void *stream);

/*
 * dls_count_sb_range -- the same over the diagonal workunits [diag_begin,
 * diag_end) of dls_split(n, symmetric, 1, diag depth) (diag_end < 0: to the end),
 * so that long runs (e.g. n = 9) can be split and resumed; the totals of all
 * ranges add up to dls_count_sb's.
 */
int dls_count_sb_range(int n, int symmetric, int64_t diag_begin, int64_t diag_end,
                       uint64_t *out_total, uint64_t *out_hourglasses, uint64_t *out_classes,
                       uint64_t *out_nodes, void *stream);

/*
 * dls_count_cells -- number of consistent assignments of the listed cells below
 * one partial square: e.g. the first k row-major cells of an order-n DLS with row
 * 0 fixed, N_n^k of the Monte Carlo section.  The listed diagonal cells
 * are enumerated on the host, the rest by the GPU search (virtual last level).
 *   record         host, n*n: the given cells (row 0 must be complete), 0xFF elsewhere;
 *   cells          host, n_cells distinct empty cells (i*n+j; left half if symmetric).
 *   out_total / out_nodes   host.
 * Synchronous.  Returns DLS_OK or a DLS_E_* code.
 */
int dls_count_cells(int n, int symmetric, const uint8_t *record, const int32_t *cells,
                    int n_cells, uint64_t *out_total, uint64_t *out_nodes, void *stream);

/*
 * dls_random_prefix -- one random descent of the Monte Carlo estimate of Section
 * 5.3: the listed empty cells of `record` are assigned in order, each
 * uniformly among its consistent values (splitmix64 stream of `seed`), into
 * out_record (host, n*n); *out_weight = product of the numbers of consistent values
 * (0 if some cell had none).  mean(weight x completions(out_record)) over
 * independent seeds is an unbiased estimate of the completions of `record`.
 * Host only.  Returns DLS_OK, DLS_E_ARG or DLS_E_PREFIX.
 */
int dls_random_prefix(int n, int symmetric, const uint8_t *record, const int32_t *cells,
                      int n_cells, uint64_t seed, uint8_t *out_record, double *out_weight);

/*
 * dls_scale_total -- the full count from the first-row-fixed count (row 0
 * is fixed "in all algorithms and experiments"; N! x the fixed count).
 * The multiplier is N! for DLS and (N/2)! * 2^(N/2) for vertically symmetric DLS
 * (a renaming keeps the symmetry only if it commutes with x -> N-1-x; DESIGN.md
 * R3); 0 for odd N with symmetric = 1.
 *   count_fixed     the count with row 0 = 0..N-1
 *   out128          host, 2 words or NULL: count_fixed * multiplier, low word first
 *   out_multiplier  host or NULL
 * Host arithmetic only (no device needed).  Returns DLS_OK or DLS_E_ARG.
 */
int dls_scale_total(int n, int symmetric, uint64_t count_fixed, uint64_t *out128, uint64_t *out_multiplier);

/*
 * dls_mc_estimate -- the Monte Carlo estimate of Section 5.3 from
 * n_samples Knuth descents (dls_random_prefix: weight w_s, completions c_s
 * counted by dls_count_cells):
 *   out[0] = mean of w_s * c_s        (unbiased estimate of the count)
 *   out[1] = its standard error       (sample standard deviation / sqrt(n); NaN for n < 2)
 *   out[2] = n_k * sum(w c) / sum(w)  (the paper's "N^k x mean completions" form;
 *                                      n_k = number of consistent k-cell prefixes)
 *   out[3] = sum(w c) / sum(w)        (weighted mean completions per prefix)
 * weights, counts: host arrays of n_samples; out: host, 4 doubles.
 * Host arithmetic only.  Returns DLS_OK or DLS_E_ARG.
 */
int dls_mc_estimate(const double *weights, const uint64_t *counts, int64_t n_samples, double n_k, double *out);

/*
 * dls_kernel_launches -- number of kernels dls_count / dls_count_async enqueue
 * per call (for the bench's launch count): the search kernel only.
 */
int dls_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* DLS_B200_H */
