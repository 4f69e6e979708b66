// split.cpp -- host-side prefix splitter (workunit decomposition).
//
// Enumerates every consistent assignment of plan cells [d0, d1) below a start
// grid with the bit-arithmetic loop of Alg. 4:
//   CR = Rows[i] | Columns[j] | MD | AD        (MD/AD only on the diagonals)
//   L  = AllN ^ CR, iterate b = L & -L, L &= L-1   (AllN = (1<<N)-1, reading R7)
// For vertical symmetry assigning v at (i,j) also assigns N-1-v at
// (i,N-1-j); both cells' constraints are folded into one candidate mask by
// reflecting the mirror cell's forbidden set (bit v <-> bit N-1-v).
//
// dls_split     : from the empty / first-row grid, cells [0, depth)
// dls::refine   : from given depth-d0 records, cells [d0, d1), with parent index
//                 (used by dls_count to cut few large workunits into many)
// dls::valid_record : host check of one record against a depth-d pattern
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "internal.h"

namespace {

inline uint32_t reflect(uint32_t m, int n) {
    uint32_t r = 0;
    for (int v = 0; v < n; ++v)
        if (m & (1u << v)) r |= 1u << (n - 1 - v);
    return r;
}

class Enumerator {
  public:
    Enumerator(const dls::Plan &plan, int d0, int d1) : plan_(plan), n_(plan.n), d0_(d0), d1_(d1) {
        all_n_ = (1u << n_) - 1u;
        for (int k = d0; k < d1; ++k) {
            ci_.push_back(plan.cells[k] / n_);
            cj_.push_back(plan.cells[k] % n_);
            cjm_.push_back(plan.vs ? n_ - 1 - plan.cells[k] % n_ : plan.cells[k] % n_);
        }
    }

    // Load a start grid; returns false if its assigned cells are inconsistent.
    bool load(const uint8_t *g) {
        std::memcpy(grid_, g, n_ * n_);
        std::memset(rows_, 0, sizeof(rows_));
        std::memset(cols_, 0, sizeof(cols_));
        md_ = ad_ = 0;
        for (int i = 0; i < n_; ++i)
            for (int j = 0; j < n_; ++j) {
                const uint8_t v = grid_[i * n_ + j];
                if (v == DLS_EMPTY) continue;
                if (v >= n_) return false;
                const uint32_t b = 1u << v;
                if ((rows_[i] & b) || (cols_[j] & b)) return false;
                if (i == j && (md_ & b)) return false;
                if (i + j == n_ - 1 && (ad_ & b)) return false;
                mark(i, j, b);
            }
        return true;
    }

    // Depth-first over cells [d0, d1); calls emit(grid) at depth d1 and counts,
    // per relative level, the consistent partial squares visited.
    template <class F>
    void run(F &&emit, std::vector<int64_t> *level_nodes) {
        const int depth = d1_ - d0_;
        if (depth == 0) { emit(grid_); return; }
        std::vector<uint32_t> L(depth), A(depth);
        int k = 0;
        L[0] = candidates(0);
        while (k >= 0) {
            if (L[k] == 0) {
                if (--k < 0) break;
                unassign(k, A[k]);
                continue;
            }
            const uint32_t b = L[k] & (0u - L[k]);   // isolate rightmost 1-bit
            L[k] &= L[k] - 1;                         // switch it off
            A[k] = b;
            assign(k, b);
            if (level_nodes) (*level_nodes)[k]++;
            if (k + 1 == depth) {
                emit(grid_);
                unassign(k, b);
            } else {
                ++k;
                L[k] = candidates(k);
            }
        }
    }

  private:
    void mark(int i, int j, uint32_t b) {
        rows_[i] ^= b;
        cols_[j] ^= b;
        if (i == j) md_ ^= b;
        if (i + j == n_ - 1) ad_ ^= b;
    }
    uint32_t forbidden(int i, int j) const {
        return rows_[i] | cols_[j] | (i == j ? md_ : 0u) | (i + j == n_ - 1 ? ad_ : 0u);
    }
    uint32_t candidates(int k) const {
        const int i = ci_[k], j = cj_[k];
        uint32_t cr = forbidden(i, j);
        if (plan_.vs && cjm_[k] != j) cr |= reflect(forbidden(i, cjm_[k]), n_);
        return all_n_ ^ (cr & all_n_);
    }
    void assign(int k, uint32_t b) {
        const int i = ci_[k], j = cj_[k];
        const int v = __builtin_ctz(b);
        mark(i, j, b);
        grid_[i * n_ + j] = (uint8_t)v;
        if (plan_.vs && cjm_[k] != j) {
            mark(i, cjm_[k], 1u << (n_ - 1 - v));
            grid_[i * n_ + cjm_[k]] = (uint8_t)(n_ - 1 - v);
        }
    }
    void unassign(int k, uint32_t b) {
        const int i = ci_[k], j = cj_[k];
        const int v = __builtin_ctz(b);
        mark(i, j, b);
        grid_[i * n_ + j] = DLS_EMPTY;
        if (plan_.vs && cjm_[k] != j) {
            mark(i, cjm_[k], 1u << (n_ - 1 - v));
            grid_[i * n_ + cjm_[k]] = DLS_EMPTY;
        }
    }

    const dls::Plan &plan_;
    int n_, d0_, d1_;
    uint32_t all_n_;
    std::vector<int> ci_, cj_, cjm_;
    uint8_t grid_[DLS_MAX_ORDER * DLS_MAX_ORDER];
    uint32_t rows_[DLS_MAX_ORDER], cols_[DLS_MAX_ORDER], md_, ad_;
};

}  // namespace

namespace {

int64_t refine_serial(const dls::Plan &plan, int d0, int d1, const uint8_t *in, int64_t n_in, uint8_t *out,
                      uint32_t *parent, int64_t capacity, int64_t *extra_nodes) {
    const int nn = plan.n * plan.n;
    Enumerator en(plan, d0, d1);
    std::vector<int64_t> lv(d1 - d0 + 1, 0);
    int64_t total = 0;
    for (int64_t p = 0; p < n_in; ++p) {
        if (!en.load(in + p * nn)) continue;   // inconsistent: no children
        en.run(
            [&](const uint8_t *g) {
                if (total < capacity) {
                    std::memcpy(out + total * nn, g, nn);
                    if (parent) parent[total] = (uint32_t)p;
                }
                ++total;
            },
            &lv);
    }
    if (extra_nodes) {
        // partial squares at depths d0+1 .. d1 (the new records included) are
        // search nodes of the original workunits that lie above the new records
        int64_t s = 0;
        for (int k = 0; k < d1 - d0; ++k) s += lv[k];
        *extra_nodes = s;
    }
    return total;
}

int host_threads() {
    if (const char *e = getenv("DLS_HOST_THREADS")) return std::max(1, atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min(32u, std::max(1u, hc));
}

}  // namespace

namespace dls {

// Multi-threaded: contiguous chunks of the input records are enumerated by
// different threads (a counting pass, then a filling pass at the chunk offsets),
// so the output order is exactly the serial one.  With too few input records the
// first level is expanded serially to make enough roots.
int64_t refine(const Plan &plan, int d0, int d1, const uint8_t *in, int64_t n_in, uint8_t *out,
               uint32_t *parent, int64_t capacity, int64_t *extra_nodes) {
    const int T = host_threads();
    const int nn = plan.n * plan.n;
    if (T <= 1 || d1 - d0 < 2 || n_in == 0)
        return refine_serial(plan, d0, d1, in, n_in, out, parent, capacity, extra_nodes);
    if (n_in < 16 * T) {
        // expand one level to get more roots (their parents map back to `in`)
        const int64_t r = refine_serial(plan, d0, d0 + 1, in, n_in, nullptr, nullptr, 0, nullptr);
        std::vector<uint8_t> roots((size_t)std::max<int64_t>(r, 1) * nn);
        std::vector<uint32_t> rpar((size_t)std::max<int64_t>(r, 1));
        refine_serial(plan, d0, d0 + 1, in, n_in, roots.data(), rpar.data(), r, nullptr);
        std::vector<uint32_t> par2;
        if (parent && capacity > 0) par2.resize((size_t)capacity);
        int64_t extra2 = 0;
        const int64_t total = refine(plan, d0 + 1, d1, roots.data(), r, out, parent ? par2.data() : nullptr,
                                     capacity, extra_nodes ? &extra2 : nullptr);
        if (parent)
            for (int64_t i = 0; i < std::min(total, capacity); ++i) parent[i] = rpar[par2[(size_t)i]];
        if (extra_nodes) *extra_nodes = r + extra2;
        return total;
    }
    const int chunks = (int)std::min<int64_t>(n_in, 4 * T);
    std::vector<int64_t> lo(chunks + 1), cnt(chunks, 0), ext(chunks, 0);
    for (int c = 0; c <= chunks; ++c) lo[c] = n_in * c / chunks;
    auto run = [&](bool fill, const std::vector<int64_t> &off) {
        std::vector<std::thread> th;
        std::atomic<int> next(0);
        for (int t = 0; t < T; ++t)
            th.emplace_back([&]() {
                for (int c = next++; c < chunks; c = next++) {
                    if (!fill) {
                        cnt[c] = refine_serial(plan, d0, d1, in + lo[c] * nn, lo[c + 1] - lo[c], nullptr, nullptr, 0,
                                               &ext[c]);
                    } else {
                        const int64_t o = off[c];
                        const int64_t room = std::max<int64_t>(0, std::min(cnt[c], capacity - o));
                        if (room <= 0) continue;
                        uint32_t *pp = parent ? parent + o : nullptr;
                        refine_serial(plan, d0, d1, in + lo[c] * nn, lo[c + 1] - lo[c], out + o * nn, pp, room,
                                      nullptr);
                        if (pp)
                            for (int64_t i = 0; i < room; ++i) pp[i] += (uint32_t)lo[c];
                    }
                }
            });
        for (auto &x : th) x.join();
    };
    run(false, {});
    std::vector<int64_t> off(chunks + 1, 0);
    for (int c = 0; c < chunks; ++c) off[c + 1] = off[c] + cnt[c];
    const int64_t total = off[chunks];
    if (out && capacity > 0) run(true, off);
    if (extra_nodes) {
        int64_t e = 0;
        for (int c = 0; c < chunks; ++c) e += ext[c];
        *extra_nodes = e;
    }
    return total;
}

bool valid_record(const Plan &plan, int depth, const uint8_t *rec) {
    const int n = plan.n;
    bool want[DLS_MAX_ORDER * DLS_MAX_ORDER] = {};
    for (int c = 0; c < n * n; ++c) want[c] = plan.pre[c] != 0;
    for (int s = 0; s < depth; ++s) {
        const int c = plan.cells[s];
        want[c] = true;
        if (plan.vs) want[(c / n) * n + (n - 1 - c % n)] = true;
    }
    for (int c = 0; c < n * n; ++c)
        if ((rec[c] != DLS_EMPTY) != want[c]) return false;
    if (plan.vs)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (rec[i * n + j] != DLS_EMPTY && rec[i * n + (n - 1 - j)] != n - 1 - rec[i * n + j])
                    return false;
    Enumerator en(plan, depth, depth);
    return en.load(rec);
}

}  // namespace dls

extern "C" int64_t dls_split(int n, int symmetric, int fixed_first_row, int depth,
                             uint8_t *out_prefixes, int64_t capacity) {
    dls::Plan plan;
    if (!dls::make_plan(n, symmetric, fixed_first_row, &plan)) {
        dls::set_error("dls_split: unsupported (n, symmetric, fixed_first_row)");
        return DLS_E_ARG;
    }
    if (depth < 0 || depth > (int)plan.cells.size() || capacity < 0 ||
        (capacity > 0 && !out_prefixes)) {
        dls::set_error("dls_split: bad depth / capacity");
        return DLS_E_ARG;
    }
    uint8_t root[DLS_MAX_ORDER * DLS_MAX_ORDER];
    std::memset(root, DLS_EMPTY, sizeof(root));
    if (fixed_first_row)
        for (int j = 0; j < n; ++j) root[j] = (uint8_t)j;
    return dls::refine(plan, 0, depth, root, 1, out_prefixes, nullptr, capacity, nullptr);
}

extern "C" int64_t dls_refine(int n, int symmetric, int fixed_first_row, int depth, const uint8_t *in,
                              int64_t n_in, int depth2, uint8_t *out, uint32_t *parent, int64_t capacity) {
    dls::Plan plan;
    if (!dls::make_plan(n, symmetric, fixed_first_row, &plan)) {
        dls::set_error("dls_refine: unsupported (n, symmetric, fixed_first_row)");
        return DLS_E_ARG;
    }
    if (depth < 0 || depth2 < depth || depth2 > (int)plan.cells.size() || n_in < 0 || (n_in > 0 && !in) ||
        capacity < 0 || (capacity > 0 && !out)) {
        dls::set_error("dls_refine: bad depth / sizes");
        return DLS_E_ARG;
    }
    for (int64_t p = 0; p < n_in; ++p)
        if (!dls::valid_record(plan, depth, in + p * n * n)) {
            dls::set_error("dls_refine: record is not a consistent depth-d prefix");
            return DLS_E_PREFIX;
        }
    return dls::refine(plan, depth, depth2, in, n_in, out, parent, capacity, nullptr);
}

// Random descent for the Monte Carlo estimate of Section 5.3: the
// cells are assigned in the given order, each uniformly among its consistent
// values (counter-based splitmix64 stream of `seed`); *out_weight = product of
// the numbers of consistent values met (0 at a dead end).  E[weight x completions]
// over the descent = number of completions of `record` (Knuth's estimator).
extern "C" int dls_random_prefix(int n, int symmetric, const uint8_t *record, const int32_t *cells, int n_cells,
                                 uint64_t seed, uint8_t *out_record, double *out_weight) {
    if (n < 1 || n > DLS_MAX_ORDER || (symmetric && n % 2) || !record || !out_record || !out_weight || n_cells < 0 ||
        (n_cells && !cells)) {
        dls::set_error("dls_random_prefix: bad arguments");
        return DLS_E_ARG;
    }
    const int nn = n * n;
    uint8_t g[DLS_MAX_ORDER * DLS_MAX_ORDER];
    std::memcpy(g, record, nn);
    uint32_t rows[DLS_MAX_ORDER] = {}, cols[DLS_MAX_ORDER] = {}, md = 0, ad = 0;
    for (int c = 0; c < nn; ++c) {
        const uint8_t v = g[c];
        if (v == DLS_EMPTY) continue;
        if (v >= n) { dls::set_error("dls_random_prefix: bad value"); return DLS_E_PREFIX; }
        const int i = c / n, j = c % n;
        const uint32_t b = 1u << v;
        if ((rows[i] & b) || (cols[j] & b) || (i == j && (md & b)) || (i + j == n - 1 && (ad & b))) {
            dls::set_error("dls_random_prefix: inconsistent record");
            return DLS_E_PREFIX;
        }
        rows[i] |= b; cols[j] |= b;
        if (i == j) md |= b;
        if (i + j == n - 1) ad |= b;
    }
    uint64_t ctr = seed * 0x9E3779B97F4A7C15ull;
    auto next = [&]() {   // splitmix64
        uint64_t z = (ctr += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    const uint32_t all_n = (1u << n) - 1u;
    double w = 1.0;
    for (int k = 0; k < n_cells; ++k) {
        const int c = cells[k], i = c / n, j = c % n;
        if (c < 0 || c >= nn || g[c] != DLS_EMPTY) { dls::set_error("dls_random_prefix: bad cell"); return DLS_E_ARG; }
        const int jm = n - 1 - j;
        uint32_t cr = rows[i] | cols[j] | (i == j ? md : 0u) | (i + j == n - 1 ? ad : 0u);
        uint32_t cand = all_n & ~cr;
        if (symmetric && jm != j) {   // the mirror cell takes n-1-v
            uint32_t ok = 0;
            for (int v = 0; v < n; ++v)
                if ((cand >> v) & 1u) {
                    const uint32_t m = 1u << (n - 1 - v);
                    const bool free = !(rows[i] & m) && !(cols[jm] & m) && !(i == jm && (md & m)) &&
                                      !(i + jm == n - 1 && (ad & m)) && (n - 1 - v) != v;
                    if (free) ok |= 1u << v;
                }
            cand = ok;
        }
        const int m = __builtin_popcount(cand);
        if (m == 0) { *out_weight = 0.0; std::memcpy(out_record, g, nn); return DLS_OK; }
        w *= m;
        int pick = (int)(next() % (uint64_t)m);
        uint32_t b = cand;
        while (pick--) b &= b - 1;
        b &= 0u - b;
        const int v = __builtin_ctz(b);
        g[c] = (uint8_t)v;
        rows[i] |= b; cols[j] |= b;
        if (i == j) md |= b;
        if (i + j == n - 1) ad |= b;
        if (symmetric && jm != j) {
            const uint32_t mb = 1u << (n - 1 - v);
            g[i * n + jm] = (uint8_t)(n - 1 - v);
            rows[i] |= mb; cols[jm] |= mb;
            if (i == jm) md |= mb;
            if (i + jm == n - 1) ad |= mb;
        }
    }
    *out_weight = w;
    std::memcpy(out_record, g, nn);
    return DLS_OK;
}
