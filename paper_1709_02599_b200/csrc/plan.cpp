// plan.cpp -- the cell order of Section 2.3 and its C ABI entry.
//
// "On each iteration step we choose the cell that has the largest V_{i,j}^k ...
//  If several cells have the same value of V, we choose the first of them when
//  ordered in lexicographic order" and "if after choosing a new cell ...
//  the number of assigned cells in some row, column, main diagonal or main
//  antidiagonal becomes N-1, then the remaining cell is automatically assigned
//  next".  Units are examined rows, columns, main diagonal, antidiagonal
//  (reading R5; this reproduces all 72 steps of Fig. 1).
//
// The planner only tracks how many cells of each unit are assigned (never
// values), as the paper prescribes.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.h"

namespace dls {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string &msg) { g_err = msg; }
const char *get_error() { return g_err.c_str(); }

bool valid_problem(int n, int symmetric, int fixed_first_row) {
    if (n < 1 || n > DLS_MAX_ORDER) return false;
    if (symmetric != 0 && symmetric != 1) return false;
    if (fixed_first_row != 0 && fixed_first_row != 1) return false;
    if (symmetric && (n % 2) != 0) return false;  // vertical symmetry needs even n (DESIGN R6)
    return true;
}

bool make_plan_from(int n, bool vs, const uint8_t *pre, const std::vector<int> &head, Plan *out) {
    if (n < 1 || n > DLS_MAX_ORDER || (vs && (n % 2) != 0)) return false;
    Plan p;
    p.n = n;
    p.vs = vs;
    p.pre.assign(pre, pre + n * n);
    p.fixed_first_row = true;
    for (int j = 0; j < n; ++j) p.fixed_first_row = p.fixed_first_row && pre[j];

    bool taken[DLS_MAX_ORDER][DLS_MAX_ORDER] = {};
    int in_row[DLS_MAX_ORDER] = {}, in_col[DLS_MAX_ORDER] = {};
    int in_md = 0, in_ad = 0;
    int assigned = 0;
    auto take = [&](int i, int j) {
        if (taken[i][j]) return;
        taken[i][j] = true;
        in_row[i]++;
        in_col[j]++;
        if (i == j) in_md++;
        if (i + j == n - 1) in_ad++;
        assigned++;
    };
    for (int c = 0; c < n * n; ++c)
        if (pre[c]) take(c / n, c % n);
    const int pre_count = assigned;
    // cells the caller wants first (e.g. a hourglass: diagonals, then row N-1)
    for (int c : head) {
        int i = c / n, j = c % n;
        if (vs && 2 * j > n - 1) j = n - 1 - j;
        if (taken[i][j]) continue;
        take(i, j);
        if (vs) take(i, n - 1 - j);
        p.cells.push_back(i * n + j);
        p.forced.push_back(0);
    }
    const int total = n * n;
    while (assigned < total) {
        int pi = -1, pj = -1;
        bool forced = false;
        // forced-cell rule: first unit with exactly n-1 assigned cells
        for (int i = 0; i < n && pi < 0; ++i)
            if (in_row[i] == n - 1)
                for (int j = 0; j < n; ++j)
                    if (!taken[i][j]) { pi = i; pj = j; break; }
        for (int j = 0; j < n && pi < 0; ++j)
            if (in_col[j] == n - 1)
                for (int i = 0; i < n; ++i)
                    if (!taken[i][j]) { pi = i; pj = j; break; }
        if (pi < 0 && in_md == n - 1)
            for (int k = 0; k < n; ++k)
                if (!taken[k][k]) { pi = k; pj = k; break; }
        if (pi < 0 && in_ad == n - 1)
            for (int k = 0; k < n; ++k)
                if (!taken[k][n - 1 - k]) { pi = k; pj = n - 1 - k; break; }
        forced = pi >= 0;
        if (!forced) {
            // V-score rule; strict '>' keeps the lexicographically first
            int best = -1;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) {
                    if (taken[i][j] || (vs && 2 * j > n - 1)) continue;
                    int v = in_row[i] + in_col[j] + (i == j ? in_md : 0) + (i + j == n - 1 ? in_ad : 0);
                    if (v > best) { best = v; pi = i; pj = j; }
                }
        }
        if (pi < 0) break;
        if (vs && 2 * pj > n - 1) pj = n - 1 - pj;  // plan the left-half representative
        take(pi, pj);
        if (vs && pj != n - 1 - pj) take(pi, n - 1 - pj);
        p.cells.push_back(pi * n + pj);
        p.forced.push_back(forced ? 1 : 0);
    }
    (void)pre_count;

    // diag depth: first prefix length after which every diagonal cell is assigned
    int remaining = 0;
    bool diag_cell[DLS_MAX_ORDER][DLS_MAX_ORDER] = {};
    for (int k = 0; k < n; ++k) diag_cell[k][k] = diag_cell[k][n - 1 - k] = true;
    bool done[DLS_MAX_ORDER][DLS_MAX_ORDER] = {};
    for (int c = 0; c < n * n; ++c)
        if (pre[c]) done[c / n][c % n] = true;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (diag_cell[i][j] && !done[i][j]) remaining++;
    p.diag_depth = 0;
    for (size_t s = 0; s < p.cells.size() && remaining > 0; ++s) {
        int i = p.cells[s] / n, j = p.cells[s] % n;
        int js[2] = {j, n - 1 - j};
        int m = (vs && j != n - 1 - j) ? 2 : 1;
        for (int t = 0; t < m; ++t)
            if (diag_cell[i][js[t]] && !done[i][js[t]]) { done[i][js[t]] = true; remaining--; }
        p.diag_depth = (int)s + 1;
    }
    *out = std::move(p);
    return true;
}

bool make_plan(int n, bool vs, bool fixed_first_row, Plan *out) {
    if (!valid_problem(n, vs, fixed_first_row)) return false;
    uint8_t pre[DLS_MAX_ORDER * DLS_MAX_ORDER] = {};
    if (fixed_first_row)
        for (int j = 0; j < n; ++j) pre[j] = 1;
    return make_plan_from(n, vs, pre, {}, out);
}

bool make_hourglass_plan(int n, bool vs, Plan *out) {
    // Section 4.3: "the first row is fixed beforehand, and the diagonals are
    // filled before everything else. Thus to produce hourglass designs we need only
    // to fill the last row of cells right after filling diagonals."
    Plan base;
    if (!make_plan(n, vs, true, &base)) return false;
    std::vector<int> head(base.cells.begin(), base.cells.begin() + base.diag_depth);
    for (int j = 0; j < n; ++j) head.push_back((n - 1) * n + j);
    uint8_t pre[DLS_MAX_ORDER * DLS_MAX_ORDER] = {};
    for (int j = 0; j < n; ++j) pre[j] = 1;
    if (!make_plan_from(n, vs, pre, head, out)) return false;
    // number of head cells actually planned (row N-1 minus its diagonal cells)
    int k = 0;
    for (int c : out->cells) {
        bool in_head = false;
        for (int h : head) in_head = in_head || h == c;
        if (!in_head) break;
        ++k;
    }
    out->hourglass_depth = k;
    return true;
}

}  // namespace dls

extern "C" int dls_plan(int n, int symmetric, int fixed_first_row, int32_t *out_cells,
                        uint8_t *out_forced, int32_t *out_n_steps, int32_t *out_diag_depth) {
    dls::Plan p;
    if (!out_cells || !out_n_steps) { dls::set_error("dls_plan: null output"); return DLS_E_ARG; }
    if (!dls::make_plan(n, symmetric, fixed_first_row, &p)) {
        dls::set_error("dls_plan: unsupported (n, symmetric, fixed_first_row)");
        return DLS_E_ARG;
    }
    for (size_t s = 0; s < p.cells.size(); ++s) {
        out_cells[s] = p.cells[s];
        if (out_forced) out_forced[s] = p.forced[s];
    }
    *out_n_steps = (int32_t)p.cells.size();
    if (out_diag_depth) *out_diag_depth = p.diag_depth;
    return DLS_OK;
}

extern "C" const char *dls_last_error(void) { return dls::get_error(); }

extern "C" int dls_scale_total(int n, int symmetric, uint64_t count_fixed, uint64_t *out128, uint64_t *out_multiplier) {
    if (n < 1 || n > DLS_MAX_ORDER) { dls::set_error("dls_scale_total: order out of range"); return DLS_E_ARG; }
    uint64_t m = 1;
    if (symmetric) {
        if (n % 2) {
            m = 0;                                   // no vertically symmetric square of odd order (R6)
        } else {
            for (int k = 2; k <= n / 2; ++k) m *= (uint64_t)k;      // (N/2)!
            m <<= n / 2;                                            // * 2^(N/2)
        }
    } else {
        for (int k = 2; k <= n; ++k) m *= (uint64_t)k;              // N!
    }
    if (out_multiplier) *out_multiplier = m;
    if (out128) {
        const unsigned __int128 p = (unsigned __int128)count_fixed * (unsigned __int128)m;
        out128[0] = (uint64_t)p;
        out128[1] = (uint64_t)(p >> 64);
    }
    return DLS_OK;
}

extern "C" int dls_mc_estimate(const double *weights, const uint64_t *counts, int64_t n_samples, double n_k, double *out) {
    if (!weights || !counts || !out || n_samples < 1) { dls::set_error("dls_mc_estimate: bad arguments"); return DLS_E_ARG; }
    long double sw = 0, swc = 0;
    for (int64_t s = 0; s < n_samples; ++s) {
        sw += weights[s];
        swc += (long double)weights[s] * (long double)counts[s];
    }
    const long double mean = swc / n_samples;
    long double ss = 0;
    for (int64_t s = 0; s < n_samples; ++s) {
        const long double d = (long double)weights[s] * (long double)counts[s] - mean;
        ss += d * d;
    }
    out[0] = (double)mean;
    out[1] = n_samples > 1 ? (double)sqrtl(ss / (n_samples - 1) / n_samples) : __builtin_nan("");
    out[2] = sw > 0 ? (double)(n_k * swc / sw) : 0.0;
    out[3] = sw > 0 ? (double)(swc / sw) : 0.0;
    return DLS_OK;
}
