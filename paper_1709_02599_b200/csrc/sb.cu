// sb.cu -- symmetry breaking with hourglass designs (Section 4).
//
// Alg. 6: generate every hourglass design (row 0 fixed, both
// diagonals, row N-1), keep those equal to their canonic form under the
// M-transformations (Alg. 5), count the diagonal Latin squares that
// complete each canonic design and weight the count by the size of its class
// (Proposition 1 / Corollary 1).
//
// On the B200:
//  * hourglass_kernel: one thread per diagonal workunit (first row + both
//    diagonals, the records of dls_split at the diagonal depth) enumerates the
//    completions of row N-1 below it and canonises every resulting hourglass;
//  * canonisation: an image under (sigma, mirror) is computed directly from the
//    three value vectors D (main diagonal), A (antidiagonal) and B (row N-1), kept
//    as 4-bit fields of 64-bit registers; the lexicographic key of a design
//    (rows top to bottom, left to right, over its assigned cells) is a
//    128-bit integer, so "image < design" is one integer comparison;
//  * class size by orbit-stabilizer: |G| / #{g : g(H) = H}, which equals Alg. 5's
//    "number of distinct designs in EQC" because the transformations form a group
//    (the oracle counts the distinct images explicitly);
//  * canonic designs are appended to a device buffer (one atomic per design) and
//    counted by the standard search kernel under the hourglass plan
//    (dls::make_hourglass_plan); the weighted sum is formed on the host.
//
// Group: sigma permutes the symmetric index pairs
// {k, N-1-k}: pair 0 (rows 0 and N-1) stays in place (row 0 may only go to row
// N-1), pairs 1..h-1 are permuted ((h-1)! ways), every pair may be swapped (2^h);
// the columns follow sigma, optionally mirrored (x2; left out for vertically
// symmetric squares, where the mirror is neutralised).  |G| = 192 for N = 8, 9,
// 768 for vertically symmetric N = 10.
#include <cuda_runtime.h>

#include <mutex>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"

namespace {

typedef unsigned long long u64;

// DLS_TIMING=1: phase times of the symmetry-broken driver on stderr
struct PhaseTimer {
    bool on = getenv("DLS_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what, cudaStream_t s) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[dls_count_sb] %-28s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

constexpr int kMaxGroup = 1536;        // 2 * 2^5 * 4! for N = 10
constexpr int kSbThreads = 256;

struct SbParams {
    const uint8_t *diag;               // diagonal workunits (n*n bytes each)
    long long n_diag;
    int n;
    int vs;
    int group;                         // number of transformations
    int mirror_choices;                // 2 (DLS) or 1 (VS)
    int soff;                          // offset of order n's sigma tables
    int k_last;                        // free left-half cells of row N-1 (planned)
    uint8_t last_cols[16];             // their columns, in plan order
    uint8_t *out_rec;                  // canonic hourglasses (n*n bytes each)
    uint32_t *out_mult;                // their class sizes
    unsigned long long *counters;      // [0] hourglasses, [1] canonic, [2] overflow
    long long capacity;
};

// Internal invariants of the checked build (-DDLS_CHECKS): bit 8 + k of
// counters[2] (bit 0 = canonic-buffer overflow); compiled out otherwise.
#ifdef DLS_CHECKS
#define SB_CHECK(cond, k) do { if (!(cond)) atomicOr(p.counters + 2, 1ull << (8 + (k))); } while (0)
#else
#define SB_CHECK(cond, k) do { } while (0)
#endif

// The sigma tables of every order n = 3..10 (2^h (h-1)! entries each, h = n/2),
// one after another: uploaded once per device and never rewritten, so calls on
// different streams or threads can never see another order's group.
constexpr int kSigmaTotal = 2 + 4 + 4 + 16 + 16 + 96 + 96 + 768;
__constant__ u64 c_sigma[kSigmaTotal];       // sigma as 4-bit fields (index -> image index)
__constant__ u64 c_sigma_inv[kSigmaTotal];

__device__ __forceinline__ int nib(u64 w, int i) { return (int)((w >> (4 * i)) & 15ull); }

// Lexicographic key of the image of (D, A, B) under (sigma, mirror), 4 bits per
// assigned cell, most significant first: rows 1..N-2 (their diagonal cells left to
// right), then row N-1.  Returned as (hi, lo) = first 16 cells, remaining cells.
__device__ void image_key(int n, u64 D, u64 A, u64 B, u64 sg, u64 si, int mirror, u64 &hi, u64 &lo) {
    // tau: column map (sigma, optionally mirrored); tau^-1(c) = si(mirror ? n-1-c : c)
    const int src0 = nib(si, 0);            // row of H that becomes row 0 (0 or n-1)
    const int srcL = nib(si, n - 1);        // row of H that becomes row n-1
    // renaming so that the image's row 0 reads 0..n-1
    u64 ren = 0;
    for (int y = 0; y < n; ++y) {
        const int ty = mirror ? n - 1 - nib(sg, y) : nib(sg, y);   // tau(y)
        const int x = src0 == 0 ? y : nib(B, y);                   // H[src0][y]
        ren |= (u64)ty << (4 * x);
    }
    int k = 0;
    hi = lo = 0;
    auto put = [&](int v) {
        const u64 r = (u64)nib(ren, v);
        if (k < 16) hi |= r << (4 * (15 - k));
        else lo |= r << (4 * (15 - (k - 16)));
        ++k;
    };
    for (int r = 1; r < n - 1; ++r) {
        const int s = nib(si, r);
        const int vd = mirror ? nib(A, s) : nib(D, s);   // image cell (r, r)
        const int va = mirror ? nib(D, s) : nib(A, s);   // image cell (r, n-1-r)
        if (r < n - 1 - r) { put(vd); put(va); }
        else if (r > n - 1 - r) { put(va); put(vd); }
        else put(vd);
    }
    for (int c = 0; c < n; ++c) {
        const int tc = nib(si, mirror ? n - 1 - c : c);   // tau^-1(c)
        put(srcL == n - 1 ? nib(B, tc) : tc);
    }
}

// Alg. 5: 0 if some image is lexicographically smaller (H not canonic), else the
// class size |G| / |stabiliser|.
__device__ uint32_t canonize_dab(int n, int group, int mirror_choices, int soff, u64 D, u64 A, u64 B) {
    const u64 *const sig = c_sigma + soff, *const sinv = c_sigma_inv + soff;
    u64 h0, l0;
    image_key(n, D, A, B, sig[0], sinv[0], 0, h0, l0);   // transformation 0 = identity
    uint32_t stab = 0;
    const int per_mirror = group / mirror_choices;
    for (int g = 0; g < per_mirror; ++g)
        for (int m = 0; m < mirror_choices; ++m) {
            u64 hi, lo;
            image_key(n, D, A, B, sig[g], sinv[g], m, hi, lo);
            if (hi < h0 || (hi == h0 && lo < l0)) return 0u;
            if (hi == h0 && lo == l0) ++stab;
        }
    return (uint32_t)group / stab;
}

// One thread per diagonal workunit: complete row N-1 (its free left-half cells in
// plan order; for VS the mirror cells follow), canonise every hourglass.
__global__ void __launch_bounds__(kSbThreads) hourglass_kernel(const SbParams p) {
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= p.n_diag) return;
    const int n = p.n;
    const uint8_t *rec = p.diag + w * (long long)n * n;
    // D, A from the record; row N-1's assigned cells; column / row masks
    u64 D = 0, A = 0, B = 0;
    uint32_t col[16] = {}, rowL = 0;
    SB_CHECK(p.k_last >= 0 && p.k_last <= 16 && n <= 16, 0);
    for (int i = 0; i < n; ++i) {
        D |= (u64)rec[i * n + i] << (4 * i);
        A |= (u64)rec[i * n + (n - 1 - i)] << (4 * i);
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const uint8_t v = rec[i * n + j];
            SB_CHECK(v == DLS_EMPTY || v < n, 1);
            if (v != DLS_EMPTY) col[j] |= 1u << v;
        }
    for (int j = 0; j < n; ++j) {
        const uint8_t v = rec[(n - 1) * n + j];
        if (v != DLS_EMPTY) { rowL |= 1u << v; B |= (u64)v << (4 * j); }
    }
    const uint32_t alln = (1u << n) - 1u;
    // DFS over the k free cells of row N-1 (k <= 8)
    uint32_t L[16];
    int lvl = 0;
    const int k = p.k_last;
    unsigned long long seen = 0, canon = 0;
    if (k == 0) {
        seen = 1;
        const uint32_t m = canonize_dab(n, p.group, p.mirror_choices, p.soff, D, A, B);
        if (m) canon = 1;
    } else {
        auto cand = [&](int l) {
            const int j = p.last_cols[l];
            uint32_t c = alln & ~(rowL | col[j]);
            if (p.vs) {   // the mirror cell (N-1, n-1-j) takes n-1-v: both must be free
                const int jm = n - 1 - j;
                uint32_t ok = 0;
                for (int v = 0; v < n; ++v)
                    if ((c >> v) & 1u) {
                        const int vm = n - 1 - v;
                        if (vm != v && !((rowL >> vm) & 1u) && !((col[jm] >> vm) & 1u)) ok |= 1u << v;
                    }
                c = ok;
            }
            return c;
        };
        L[0] = cand(0);
        while (lvl >= 0) {
            if (!L[lvl]) {
                --lvl;
                if (lvl >= 0) {   // unassign the value of level lvl
                    const int j = p.last_cols[lvl];
                    const int v = nib(B, j);
                    rowL &= ~(1u << v);
                    col[j] &= ~(1u << v);
                    B &= ~(15ull << (4 * j));
                    if (p.vs) {
                        const int jm = n - 1 - j, vm = n - 1 - v;
                        rowL &= ~(1u << vm);
                        col[jm] &= ~(1u << vm);
                        B &= ~(15ull << (4 * jm));
                    }
                }
                continue;
            }
            const uint32_t b = L[lvl] & (0u - L[lvl]);
            L[lvl] ^= b;
            const int v = __ffs(b) - 1;
            const int j = p.last_cols[lvl];
            rowL |= b;
            col[j] |= b;
            B |= (u64)v << (4 * j);
            if (p.vs) {
                const int jm = n - 1 - j, vm = n - 1 - v;
                rowL |= 1u << vm;
                col[jm] |= 1u << vm;
                B |= (u64)vm << (4 * jm);
            }
            if (lvl + 1 == k) {
                ++seen;
                const uint32_t m = canonize_dab(n, p.group, p.mirror_choices, p.soff, D, A, B);
                SB_CHECK(m == 0u || (uint32_t)p.group % m == 0u, 2);     // |G| / |Stab|
                if (m) {
                    ++canon;
                    const unsigned long long slot = atomicAdd(p.counters + 3, 1ull);
                    if ((long long)slot < p.capacity) {
                        uint8_t *dst = p.out_rec + slot * (unsigned long long)(n * n);
                        for (int c = 0; c < n * n; ++c) dst[c] = rec[c];
                        for (int c = 0; c < n; ++c) dst[(n - 1) * n + c] = (uint8_t)nib(B, c);
                        p.out_mult[slot] = m;
                    } else {
                        atomicOr(p.counters + 2, 1ull);
                    }
                }
                // undo the last cell at once
                rowL &= ~b;
                col[j] &= ~b;
                B &= ~(15ull << (4 * j));
                if (p.vs) {
                    const int jm = n - 1 - j, vm = n - 1 - v;
                    rowL &= ~(1u << vm);
                    col[jm] &= ~(1u << vm);
                    B &= ~(15ull << (4 * jm));
                }
            } else {
                ++lvl;
                L[lvl] = cand(lvl);
            }
        }
    }
    if (k == 0 && canon) {
        const unsigned long long slot = atomicAdd(p.counters + 3, 1ull);
        if ((long long)slot < p.capacity) {
            uint8_t *dst = p.out_rec + slot * (unsigned long long)(n * n);
            for (int c = 0; c < n * n; ++c) dst[c] = rec[c];
            p.out_mult[slot] = canonize_dab(n, p.group, p.mirror_choices, p.soff, D, A, B);
        } else {
            atomicOr(p.counters + 2, 1ull);
        }
    }
    atomicAdd(p.counters + 0, seen);
    atomicAdd(p.counters + 1, canon);
}

// Canonise given hourglass records (for tests / external drivers).
__global__ void __launch_bounds__(kSbThreads) canonize_kernel(const uint8_t *recs, long long n_rec, int n, int group,
                                                              int mirror_choices, int soff, uint32_t *out) {
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_rec) return;
    const uint8_t *rec = recs + w * (long long)n * n;
    u64 D = 0, A = 0, B = 0;
    for (int i = 0; i < n; ++i) {
        D |= (u64)rec[i * n + i] << (4 * i);
        A |= (u64)rec[i * n + (n - 1 - i)] << (4 * i);
        B |= (u64)rec[(n - 1) * n + i] << (4 * i);
    }
    out[w] = canonize_dab(n, group, mirror_choices, soff, D, A, B);
}

int fail(cudaError_t e, const char *what) {
    dls::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DLS_E_CUDA;
}

// sigma tables of order n: 2^h (h-1)! permutations of the rows/columns (pair
// {0, n-1} kept in place, the other symmetric pairs permuted, each pair swapped
// or not), identity first
void sigma_tables(int n, std::vector<u64> &sg, std::vector<u64> &si) {
    const int h = n / 2;
    std::vector<int> pi(h);
    std::iota(pi.begin(), pi.end(), 0);
    do {
        for (int s = 0; s < (1 << h); ++s) {
            int sigma[16], inv[16];
            for (int i = 0; i < n; ++i) sigma[i] = i;
            for (int i = 0; i < h; ++i) {
                const int a = pi[i];
                int lo = a, hi = n - 1 - a;
                if (s & (1 << a)) std::swap(lo, hi);
                sigma[i] = lo;
                sigma[n - 1 - i] = hi;
            }
            for (int i = 0; i < n; ++i) inv[sigma[i]] = i;
            u64 a = 0, b = 0;
            for (int i = 0; i < n; ++i) { a |= (u64)sigma[i] << (4 * i); b |= (u64)inv[i] << (4 * i); }
            sg.push_back(a);
            si.push_back(b);
        }
    } while (std::next_permutation(pi.begin() + 1, pi.end()));
}

// Offset of order n's tables in c_sigma / c_sigma_inv.
int sigma_offset(int n) {
    int off = 0;
    for (int m = 3; m < n; ++m) {
        int h = m / 2, f = 1;
        for (int k = 2; k < h; ++k) f *= k;
        off += (1 << h) * f;
    }
    return off;
}

// Upload every order's tables to the current device, once (thread-safe).
int upload_groups() {
    static std::once_flag once[64];
    static int status[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(e, "cudaGetDevice");
    std::call_once(once[dev & 63], [&]() {
        std::vector<u64> sg, si;
        for (int n = 3; n <= DLS_MAX_ORDER; ++n) sigma_tables(n, sg, si);
        cudaError_t e1 = sg.size() == (size_t)kSigmaTotal ? cudaSuccess : cudaErrorInvalidValue;
        if (e1 == cudaSuccess) e1 = cudaMemcpyToSymbol(c_sigma, sg.data(), sg.size() * sizeof(u64));
        if (e1 == cudaSuccess) e1 = cudaMemcpyToSymbol(c_sigma_inv, si.data(), si.size() * sizeof(u64));
        status[dev & 63] = (int)e1;
    });
    if (status[dev & 63] != (int)cudaSuccess) return fail((cudaError_t)status[dev & 63], "group tables");
    return DLS_OK;
}

// The transformation group of order n: |G| (sigma count x mirrors), the mirror
// choices and the tables' offset; DLS_E_CUDA if the tables could not be uploaded.
int build_group(int n, bool vs, int *mirror_choices, int *soff) {
    const int rc = upload_groups();
    if (rc) return rc;
    const int h = n / 2;
    int f = 1;
    for (int k = 2; k < h; ++k) f *= k;
    *mirror_choices = vs ? 1 : 2;
    *soff = sigma_offset(n);
    return (1 << h) * f * *mirror_choices;
}

bool device_ptr(const void *ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" int dls_canonize(int n, int symmetric, const uint8_t *hourglasses, int64_t n_rec, uint32_t *out_mult,
                            void *stream) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        dls::set_error("no CUDA device: the B200 path is the only path (no CPU fallback)");
        return DLS_E_NODEVICE;
    }
    if (n < 3 || n > DLS_MAX_ORDER || (symmetric && n % 2) || n_rec < 0 || (n_rec && (!hourglasses || !out_mult))) {
        dls::set_error("dls_canonize: bad arguments");
        return DLS_E_ARG;
    }
    if (n_rec == 0) return DLS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int mirrors = 0, soff = 0;
    const int group = build_group(n, symmetric, &mirrors, &soff);
    if (group < 0) return group;
    cudaError_t e;
    const uint8_t *d_in = hourglasses;
    uint32_t *d_out = out_mult;
    void *tmp_in = nullptr, *tmp_out = nullptr;
    const size_t bytes = (size_t)n_rec * n * n;
    if (!device_ptr(hourglasses)) {
        if ((e = dls::scratch_alloc(&tmp_in, bytes, s)) != cudaSuccess) return fail(e, "scratch_alloc");
        cudaMemcpyAsync(tmp_in, hourglasses, bytes, cudaMemcpyHostToDevice, s);
        d_in = (const uint8_t *)tmp_in;
    }
    const bool host_out = !device_ptr(out_mult);
    if (host_out) {
        if ((e = dls::scratch_alloc(&tmp_out, (size_t)n_rec * 4, s)) != cudaSuccess) {
            if (tmp_in) cudaFreeAsync(tmp_in, s);
            cudaStreamSynchronize(s);
            return fail(e, "scratch_alloc");
        }
        d_out = (uint32_t *)tmp_out;
    }
    canonize_kernel<<<(unsigned)((n_rec + kSbThreads - 1) / kSbThreads), kSbThreads, 0, s>>>(d_in, n_rec, n, group,
                                                                                             mirrors, soff, d_out);
    e = cudaGetLastError();
    if (e == cudaSuccess && host_out) e = cudaMemcpyAsync(out_mult, d_out, (size_t)n_rec * 4, cudaMemcpyDeviceToHost, s);
    if (tmp_in) cudaFreeAsync(tmp_in, s);
    if (tmp_out) cudaFreeAsync(tmp_out, s);
    const cudaError_t es = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = es;
    return e == cudaSuccess ? DLS_OK : fail(e, "dls_canonize");
}

extern "C" int dls_count_sb_range(int n, int symmetric, int64_t diag_begin, int64_t diag_end, uint64_t *out_total,
                                  uint64_t *out_hourglasses, uint64_t *out_classes, uint64_t *out_nodes,
                                  void *stream) {
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
        cudaGetLastError();
        dls::set_error("no CUDA device: the B200 path is the only path (no CPU fallback)");
        return DLS_E_NODEVICE;
    }
    dls::Plan base, hg;
    if (n < 3 || !dls::make_plan(n, symmetric, 1, &base) || !dls::make_hourglass_plan(n, symmetric, &hg)) {
        dls::set_error("dls_count_sb: unsupported order (3 <= n <= 10; even n when symmetric)");
        return DLS_E_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    PhaseTimer timer;
    const int nn = n * n;
    const int dd = base.diag_depth;
    // the hourglass plan lists the diagonal cells exactly as the standard plan
    for (int c = 0; c < dd; ++c)
        if (hg.cells[c] != base.cells[c]) { dls::set_error("dls_count_sb: plan mismatch"); return DLS_E_ARG; }
    const int hd = hg.hourglass_depth;
    SbParams sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.n = n;
    sp.vs = symmetric;
    sp.k_last = hd - dd;
    for (int l = 0; l < sp.k_last; ++l) sp.last_cols[l] = (uint8_t)(hg.cells[dd + l] % n);
    sp.group = build_group(n, symmetric, &sp.mirror_choices, &sp.soff);
    if (sp.group < 0) return sp.group;
    // diagonal workunits (host split), the range [diag_begin, diag_end) of them,
    // processed in chunks to bound memory
    const int64_t n_all = dls_split(n, symmetric, 1, dd, nullptr, 0);
    if (n_all < 0) return (int)n_all;
    if (diag_end < 0 || diag_end > n_all) diag_end = n_all;
    if (diag_begin < 0 || diag_begin > diag_end) {
        dls::set_error("dls_count_sb_range: bad range");
        return DLS_E_ARG;
    }
    std::vector<uint8_t> all((size_t)std::max<int64_t>(n_all, 1) * nn);
    dls_split(n, symmetric, 1, dd, all.data(), n_all);
    timer.mark("host split (diagonals)", s);
    const int64_t n_diag = diag_end - diag_begin;
    const uint8_t *const diag_base = all.data() + diag_begin * nn;
    const int64_t chunk = 1 << 20;
    const long long cap = 1 << 22;     // canonic hourglasses per chunk
    uint8_t *d_diag = nullptr, *d_rec = nullptr;
    uint32_t *d_mult = nullptr;
    unsigned long long *d_cnt = nullptr;
    cudaError_t e;
    auto cleanup = [&]() {
        for (void *q : {(void *)d_diag, (void *)d_rec, (void *)d_mult, (void *)d_cnt})
            if (q) cudaFreeAsync(q, s);
        cudaStreamSynchronize(s);
        dls::scratch_trim((size_t)64 << 20);   // keep the search's small scratch, not ours
    };
    // scratch from the library's stream-ordered pool
    if ((e = dls::scratch_alloc((void **)&d_diag, (size_t)std::min<int64_t>(n_diag, chunk) * nn + 1, s)) != cudaSuccess ||
        (e = dls::scratch_alloc((void **)&d_rec, (size_t)cap * nn, s)) != cudaSuccess ||
        (e = dls::scratch_alloc((void **)&d_mult, (size_t)cap * 4, s)) != cudaSuccess ||
        (e = dls::scratch_alloc((void **)&d_cnt, 4 * sizeof(unsigned long long), s)) != cudaSuccess) {
        cleanup();
        return fail(e, "cudaMalloc");
    }
    unsigned long long total = 0, hourglasses = 0, classes = 0, nodes = 0;
    std::vector<uint8_t> reps;
    std::vector<uint32_t> mult;
    std::vector<uint64_t> counts;
    for (int64_t off = 0; off < n_diag; off += chunk) {
        const int64_t m = std::min<int64_t>(chunk, n_diag - off);
        cudaMemcpyAsync(d_diag, diag_base + off * nn, (size_t)m * nn, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(d_cnt, 0, 4 * sizeof(unsigned long long), s);
        sp.diag = d_diag;
        sp.n_diag = m;
        sp.out_rec = d_rec;
        sp.out_mult = d_mult;
        sp.counters = d_cnt;
        sp.capacity = cap;
        hourglass_kernel<<<(unsigned)((m + kSbThreads - 1) / kSbThreads), kSbThreads, 0, s>>>(sp);
        if ((e = cudaGetLastError()) != cudaSuccess) { cleanup(); return fail(e, "hourglass_kernel"); }
        unsigned long long cnt[4];
        cudaMemcpyAsync(cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) { cleanup(); return fail(e, "hourglass_kernel"); }
        timer.mark("H2D + hourglass kernel", s);
        if (cnt[2] >> 8) {
            cleanup();
            dls::set_error("dls_count_sb: internal check failed (mask " + std::to_string(cnt[2] >> 8) + ")");
            return DLS_E_CUDA;
        }
        if (cnt[2]) { cleanup(); dls::set_error("dls_count_sb: canonic buffer overflow"); return DLS_E_ARG; }
        hourglasses += cnt[0];
        classes += cnt[1];
        const long long k = (long long)cnt[3];
        if (k == 0) continue;
        // count the completions of every canonic design (hourglass plan)
        counts.assign((size_t)k, 0);
        mult.resize((size_t)k);
        cudaMemcpyAsync(mult.data(), d_mult, (size_t)k * 4, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        uint64_t part = 0, nd = 0;
        // canonic designs have large, uneven subtrees: always cut them to >= ~8 records per lane
        int rc = dls::count_records(hg, hd, d_rec, k, counts.data(), &part, &nd, stream, 1200000);
        if (rc != DLS_OK) { cleanup(); return rc; }
        nodes += nd;
        for (long long i = 0; i < k; ++i) total += counts[(size_t)i] * (unsigned long long)mult[(size_t)i];
        timer.mark("refine + search canonic", s);
    }
    cleanup();
    if (out_total) *out_total = total;
    if (out_hourglasses) *out_hourglasses = hourglasses;
    if (out_classes) *out_classes = classes;
    if (out_nodes) *out_nodes = nodes;
    return DLS_OK;
}

extern "C" int dls_count_sb(int n, int symmetric, uint64_t *out_total, uint64_t *out_hourglasses,
                            uint64_t *out_classes, uint64_t *out_nodes, void *stream) {
    return dls_count_sb_range(n, symmetric, 0, -1, out_total, out_hourglasses, out_classes, out_nodes, stream);
}
