// count.cu -- the sm_100a search kernel behind dls_count / dls_count_async.
//
// What it computes: for every prefix record (a workunit of P:481) the number of
// diagonal Latin squares that complete it -- the loop nest of Alg. 1/2
// in the bit-arithmetic form of Alg. 4:
//     CR = Rows[i] | Columns[j]            (prefixes cover both diagonals, so MD/AD
//     L  = AllN ^ CR                        are already full and drop out)
//     for (; L; L &= L-1) { b = L & -L; mark b; <next cell>; unmark b; }
// and, in the vertically symmetric case, the left half only, the right
// half being derived as LS[i][N-1-j] = N-1-LS[i][j].
//
// How ("Kernel"):
//  * persistent grid, one DFS per lane; the nested loops become one iterative
//    step (descend / backtrack selected branch-free), so all busy lanes of a warp
//    execute the same instruction stream;
//  * per-level candidate sets L[] (Alg. 4's L[i][j]) live in a per-lane stack in
//    shared memory, u32 per level, layout [level][lane] (bank-conflict free);
//    the "current" L is kept in a register, and its lowest set bit is the value
//    assigned at that level, exactly as Alg. 4 keeps LS = L & -L;
//  * Rows/Columns occupancy sets are packed bit fields in 64-bit registers, so a
//    cell's candidate set is two funnel shifts and one LOP3;
//  * a global atomic work queue hands prefixes to lanes (warp-aggregated: one
//    atomic per warp refill); once it is drained, idle lanes receive the
//    untried siblings of the shallowest open level of a busy lane of their warp
//    (warp-vote donation, ballot/shuffle pairing);
//  * counts: 32-bit per K-step burst -> 64-bit per lane -> atomicAdd per prefix
//    (optional) and one 64-bit atomicAdd per block for the total.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace {

typedef unsigned long long u64;

constexpr int kMaxLevels = 100;     // n*n for n = 10
constexpr int kBlock = 256;         // threads per CTA
constexpr int kBurst = 32;          // DFS steps between warp scheduling points
constexpr int kMinDonateDepth = 6;  // do not donate subtrees shallower than this
constexpr unsigned kFull = 0xFFFFFFFFu;

struct Params {
    const uint8_t *prefixes;
    long long n_prefix;
    u64 *counts;       // per-prefix counts (may be null)
    const uint32_t *parent;  // record -> output slot (null = identity; set by refinement)
    u64 *stats;        // DLS_STATS_WORDS words, see dls_b200.h
    u64 pat[2];        // cells assigned in a prefix, bit i*n+j
    int L;             // number of searched levels (plan cells after the prefix)
    int donate;        // enable warp-level subtree donation
    uint32_t tab[kMaxLevels + 2];  // tab[l], l = 1..L: packed geometry of level l
};

// ---------------------------------------------------------------- geometry

// Row / column sets are bit fields inside W 64-bit words.  For DLS a row field
// holds the N value bits; for vertical symmetry a row field holds N/2 "pair"
// bits (a row always contains v and N-1-v together) and only the N/2 left
// columns are tracked (the right column N-1-j is the mirror of column j).
template <int N, bool VS>
struct Geo {
    static constexpr int H = N / 2;
    static constexpr int RF = VS ? (H > 0 ? H : 1) : N;        // row field width
    static constexpr int CF = N;                               // column field width
    static constexpr int NC = VS ? H : N;                      // tracked columns
    static constexpr int RPW = 64 / RF;
    static constexpr int CPW = 64 / CF;
    static constexpr int WR = (N + RPW - 1) / RPW;
    static constexpr int WC = (NC + CPW - 1) / CPW;
    static constexpr uint32_t ALLN = (1u << N) - 1u;
    static constexpr uint32_t HMASK = (1u << H) - 1u;
    // value v -> bit position used inside the kernel.  DLS: v.  VS: the mirror
    // of position p is p +- H, so that a row's pair mask expands with one IMAD.
    __host__ __device__ static constexpr int pos(int v) {
        return !VS ? v : (v < H ? v : H + (N - 1 - v));
    }
};

// tab entry: bits 0-5 row shift, bit 6 row word, bits 8-13 col shift, bit 14 col word
__host__ __device__ inline uint32_t rsh(uint32_t e) { return e & 63u; }
__host__ __device__ inline uint32_t rwd(uint32_t e) { return (e >> 6) & 1u; }
__host__ __device__ inline uint32_t csh(uint32_t e) { return (e >> 8) & 63u; }
__host__ __device__ inline uint32_t cwd(uint32_t e) { return (e >> 14) & 1u; }

template <int W>
__device__ __forceinline__ uint32_t field(const u64 (&a)[W], uint32_t sh, uint32_t wd) {
    u64 w = a[0];
    if (W == 2) w = wd ? a[W - 1] : a[0];
    return (uint32_t)(w >> sh);
}

template <int W>
__device__ __forceinline__ void flip(u64 (&a)[W], uint32_t sh, uint32_t wd, uint32_t bits) {
    const u64 t = (u64)bits << sh;
    if (W == 1) {
        a[0] ^= t;
    } else {
        a[0] ^= wd ? 0ull : t;
        a[W - 1] ^= wd ? t : 0ull;
    }
}

template <int N, bool VS>
struct Lane {
    typedef Geo<N, VS> G;
    u64 R[G::WR];
    u64 C[G::WC];

    __device__ __forceinline__ uint32_t cand(uint32_t e) const {
        uint32_t r = field<G::WR>(R, rsh(e), rwd(e));
        const uint32_t c = field<G::WC>(C, csh(e), cwd(e));
        if (VS) r = (r & G::HMASK) * ((1u << G::H) + 1u);   // pairs -> both values
        return G::ALLN & ~(r | c);
    }
    __device__ __forceinline__ void toggle(uint32_t e, uint32_t b) {
        uint32_t rb = b;
        if (VS) rb = (b | (b >> G::H)) & G::HMASK;            // value bit -> pair bit
        flip<G::WR>(R, rsh(e), rwd(e), rb);
        flip<G::WC>(C, csh(e), cwd(e), b);
    }
};

__host__ __device__ inline bool pat_bit(const u64 *pat, int c) {
    return (pat[c >> 6] >> (c & 63)) & 1ull;
}

// Build the row/column sets of one prefix record and validate it: exactly the
// pattern cells assigned, values < N, no repeated value in a row, column or
// diagonal, and (VS) mirror consistency LS[i][N-1-j] = N-1-LS[i][j].
template <int N, bool VS>
__device__ bool load_prefix(const uint8_t *__restrict__ rec, const Params &p, Lane<N, VS> &st) {
    typedef Geo<N, VS> G;
    uint32_t rm[N], cm[N], sr[N], sc[G::NC > 0 ? G::NC : 1];
    uint32_t md = 0, ad = 0;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) { rm[i] = cm[i] = sr[i] = 0; }
#pragma unroll
    for (int j = 0; j < G::NC; ++j) sc[j] = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const uint32_t v = __ldg(rec + i * N + j);
            const bool assigned = v != DLS_EMPTY;
            ok &= assigned == pat_bit(p.pat, i * N + j);
            if (assigned) {
                ok &= v < (uint32_t)N;
                const uint32_t b = 1u << (v & 31u);
                ok &= !(rm[i] & b) && !(cm[j] & b);
                rm[i] |= b;
                cm[j] |= b;
                if (i == j) { ok &= !(md & b); md |= b; }
                if (i + j == N - 1) { ok &= !(ad & b); ad |= b; }
                if (VS) {
                    const uint32_t m = __ldg(rec + i * N + (N - 1 - j));
                    ok &= m == (uint32_t)(N - 1) - v;
                    const uint32_t pb = 1u << (G::pos((int)(v & 15u)) & 31);
                    if (2 * j < N - 1) {
                        sr[i] |= (pb | (pb >> G::H)) & G::HMASK;
                        sc[j < G::NC ? j : 0] |= pb;
                    }
                } else {
                    sr[i] |= b;
                    sc[j < G::NC ? j : 0] |= b;
                }
            }
        }
    }
#pragma unroll
    for (int w = 0; w < G::WR; ++w) st.R[w] = 0;
#pragma unroll
    for (int w = 0; w < G::WC; ++w) st.C[w] = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) st.R[i / G::RPW] |= (u64)sr[i] << ((i % G::RPW) * G::RF);
#pragma unroll
    for (int j = 0; j < G::NC; ++j) st.C[j / G::CPW] |= (u64)sc[j] << ((j % G::CPW) * G::CF);
    return ok;
}

template <int W>
__device__ __forceinline__ u64 warp_sum(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
    return v;
}

template <int N, bool VS>
__global__ void __launch_bounds__(kBlock, (Geo<N, VS>::WR + Geo<N, VS>::WC > 2) ? 3 : 4)
dls_search_kernel(const __grid_constant__ Params p) {
    typedef Geo<N, VS> G;
    extern __shared__ uint32_t smem[];
    const int L = p.L;
    uint32_t *tab_s = smem;                        // L + 2 entries (padded to 4)
    uint32_t *stack = smem + ((L + 2 + 3) & ~3);   // (L + 2) slots x kBlock lanes
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const unsigned lt_mask = (1u << lane) - 1u;

    for (int l = tid; l < L + 2; l += kBlock) tab_s[l] = l <= L ? p.tab[l] : 0u;
    // slots for levels -1 and 0 are read (idle lanes, backtrack from level 1) but
    // never written: they stay 0
    stack[tid] = 0u;
    stack[kBlock + tid] = 0u;
    __syncthreads();
    // S[(l + 1) * kBlock] is the slot of level l (l = -1 .. L)
    uint32_t *const S = stack + tid;

    Lane<N, VS> st;
#pragma unroll
    for (int w = 0; w < G::WR; ++w) st.R[w] = 0;
#pragma unroll
    for (int w = 0; w < G::WC; ++w) st.C[w] = 0;
    int lvl = 0;           // 0: idle / finished, 1..L: searching level lvl
    uint32_t cur = 0;      // untried candidates at level lvl
    uint32_t ecur = tab_s[0];
    long long pid = -1;    // prefix being searched
    u64 cnt = 0;           // completions found for pid by this lane
    u64 tot = 0, steps_dn = 0, donations = 0;
    bool qempty = false;
    const u64 n_prefix = (u64)p.n_prefix;

    for (;;) {
        // ------------------------------------------------ scheduling point
        if (pid >= 0 && lvl == 0) {
            if (p.counts && cnt) atomicAdd(p.counts + (p.parent ? (long long)p.parent[pid] : pid), cnt);
            tot += cnt;
            cnt = 0;
            pid = -1;
        }
        if (!qempty) {
            const unsigned idle = __ballot_sync(kFull, pid < 0);
            if (idle) {
                const int leader = __ffs(idle) - 1;
                u64 base = 0;
                if (lane == leader) base = atomicAdd(p.stats + 3, (u64)__popc(idle));
                base = __shfl_sync(kFull, base, leader);
                if (base + (u64)__popc(idle) >= n_prefix) qempty = true;
                if (pid < 0) {
                    const u64 my = base + (u64)__popc(idle & lt_mask);
                    if (my < n_prefix) {
                        pid = (long long)my;
                        const bool ok = load_prefix<N, VS>(p.prefixes + my * (u64)(N * N), p, st);
                        if (!ok) {
                            atomicOr(p.stats + 2, 1ull);
                            lvl = 0;
                            cur = 0;
                        } else if (L == 0) {
                            cnt = 1;   // the prefix is a complete square
                            lvl = 0;
                            cur = 0;
                        } else {
                            lvl = 1;
                            ecur = tab_s[1];
                            const uint32_t c = st.cand(ecur);
                            if (L == 1) { cnt += __popc(c); cur = 0; } else { cur = c; }
                        }
                    }
                }
            }
        }
        if (qempty) {
            const unsigned idle = __ballot_sync(kFull, pid < 0);
            if (idle == kFull) break;
            if (idle && p.donate) {
                // ---- warp-vote donation: busy lanes with an open level give the
                // untried siblings of their shallowest open level to idle lanes.
                int split = 0;
                uint32_t rest = 0;
                if (pid >= 0 && lvl > 0) {
                    for (int l = 1; l < lvl && l <= L - kMinDonateDepth; ++l) {
                        const uint32_t s = S[(l + 1) * kBlock];
                        if (s & (s - 1u)) { split = l; rest = s & (s - 1u); break; }
                    }
                    if (!split && lvl <= L - kMinDonateDepth && (cur & (cur - 1u))) {
                        split = lvl;
                        rest = cur & (cur - 1u);   // keep the lowest for ourselves
                    }
                }
                const unsigned donors = __ballot_sync(kFull, split > 0);
                const int pairs = min(__popc(donors), __popc(idle));
                if (pairs) {
                    // k-th idle lane <- k-th donor lane
                    const int my_rank = __popc(idle & lt_mask);
                    int src = 0;
                    if (pid < 0 && my_rank < pairs) src = __fns(donors, 0, my_rank + 1);
                    const int dn_rank = __popc(donors & lt_mask);
                    const int d_split = __shfl_sync(kFull, split, src);
                    const uint32_t d_rest = __shfl_sync(kFull, rest, src);
                    const long long d_pid = __shfl_sync(kFull, pid, src);
                    const bool recv = pid < 0 && my_rank < pairs;
                    const bool give = split > 0 && dn_rank < pairs;
                    if (recv) {
                        // copy the donor's path above the split level
                        uint32_t *const Sd = stack + (tid - lane + src);
                        for (int l = 1; l < d_split; ++l) S[(l + 1) * kBlock] = Sd[(l + 1) * kBlock];
                    }
                    __syncwarp();
                    if (give) {
                        if (split < lvl) S[(split + 1) * kBlock] &= 0u - S[(split + 1) * kBlock];
                        else cur &= 0u - cur;
                        ++donations;
                    }
                    if (recv) {
                        pid = d_pid;
                        load_prefix<N, VS>(p.prefixes + (u64)pid * (u64)(N * N), p, st);
                        for (int l = 1; l < d_split; ++l) {
                            const uint32_t s = S[(l + 1) * kBlock];
                            st.toggle(tab_s[l], s & (0u - s));
                        }
                        lvl = d_split;
                        ecur = tab_s[d_split];
                        cur = d_rest;
                        cnt = 0;
                    }
                }
            }
        }

        // ------------------------------------------------ kBurst DFS steps
        uint32_t cnt32 = 0, dn32 = 0;
#pragma unroll 4
        for (int s = 0; s < kBurst; ++s) {
            const bool dn = cur != 0u;
            const uint32_t b = cur & (0u - cur);          // isolate rightmost 1-bit
            const int nl = max(dn ? lvl + 1 : lvl - 1, 0);
            const uint32_t en = tab_s[nl];
            const uint32_t sp = S[lvl * kBlock];          // slot of level lvl-1
            if (dn) S[(lvl + 1) * kBlock] = cur;           // push L of level lvl (b = lowest)
            const uint32_t bb = sp & (0u - sp);           // value assigned at lvl-1
            st.toggle(dn ? ecur : en, dn ? b : bb);        // mark b / unmark bb (Alg. 4 XOR)
            const uint32_t c = st.cand(en);                // AllN ^ (Rows | Columns)
            const bool leaf = nl == L;
            const uint32_t pc = leaf ? (uint32_t)__popc(c) : 0u;
            cnt32 += pc;
            dn32 += dn ? 1u : 0u;
            cur = dn ? (leaf ? 0u : c) : (sp ^ bb);       // L &= L-1 on the way back
            lvl = nl;
            ecur = en;
        }
        cnt += cnt32;
        steps_dn += dn32;
    }

    // ------------------------------------------------ block reduction, 1 atomic per block
    __shared__ u64 red[3][kBlock / 32];
    tot = warp_sum<1>(tot);
    steps_dn = warp_sum<1>(steps_dn);
    donations = warp_sum<1>(donations);
    if (lane == 0) {
        red[0][tid >> 5] = tot;
        red[1][tid >> 5] = steps_dn;
        red[2][tid >> 5] = donations;
    }
    __syncthreads();
    if (tid == 0) {
        u64 a = 0, b = 0, c = 0;
        for (int w = 0; w < kBlock / 32; ++w) { a += red[0][w]; b += red[1][w]; c += red[2][w]; }
        atomicAdd(p.stats + 0, a);
        atomicAdd(p.stats + 1, b);
        atomicAdd(p.stats + 4, c);
    }
}

typedef void (*KernelFn)(Params);

template <int N, bool VS>
KernelFn kernel_for() { return dls_search_kernel<N, VS>; }

KernelFn pick_kernel(int n, bool vs) {
    switch (n) {
        case 1: return kernel_for<1, false>();
        case 2: return vs ? kernel_for<2, true>() : kernel_for<2, false>();
        case 3: return kernel_for<3, false>();
        case 4: return vs ? kernel_for<4, true>() : kernel_for<4, false>();
        case 5: return kernel_for<5, false>();
        case 6: return vs ? kernel_for<6, true>() : kernel_for<6, false>();
        case 7: return kernel_for<7, false>();
        case 8: return vs ? kernel_for<8, true>() : kernel_for<8, false>();
        case 9: return kernel_for<9, false>();
        case 10: return vs ? kernel_for<10, true>() : kernel_for<10, false>();
        default: return nullptr;
    }
}

// host mirror of Geo<> for building tab entries
void field_geometry(int n, bool vs, int *rf, int *rpw, int *cf, int *cpw) {
    const int h = n / 2;
    *rf = vs ? (h > 0 ? h : 1) : n;
    *cf = n;
    *rpw = 64 / *rf;
    *cpw = 64 / *cf;
}

int cuda_fail(cudaError_t e, const char *what) {
    dls::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DLS_E_CUDA;
}

// Everything a launch needs that depends only on (n, vs, fixed_first_row, depth).
int prepare(int n, int symmetric, int fixed_first_row, int depth, Params *prm) {
    dls::Plan plan;
    if (!dls::make_plan(n, symmetric, fixed_first_row, &plan)) {
        dls::set_error("dls_count: unsupported (n, symmetric, fixed_first_row)");
        return DLS_E_ARG;
    }
    const int steps = (int)plan.cells.size();
    if (depth < plan.diag_depth || depth > steps) {
        dls::set_error("dls_count: depth must satisfy diag_depth <= depth <= n_steps");
        return DLS_E_ARG;
    }
    std::memset(prm, 0, sizeof(*prm));
    prm->L = steps - depth;
    int rf, rpw, cf, cpw;
    field_geometry(n, symmetric, &rf, &rpw, &cf, &cpw);
    for (int l = 1; l <= prm->L; ++l) {
        const int cell = plan.cells[depth + l - 1];
        const int i = cell / n, j = cell % n;
        const uint32_t e = (uint32_t)((i % rpw) * rf) | ((uint32_t)(i / rpw) << 6) |
                           ((uint32_t)((j % cpw) * cf) << 8) | ((uint32_t)(j / cpw) << 14);
        prm->tab[l] = e;
    }
    // assigned-cell pattern of a depth-`depth` prefix
    auto set = [&](int c) { prm->pat[c >> 6] |= 1ull << (c & 63); };
    if (fixed_first_row)
        for (int j = 0; j < n; ++j) set(j);
    for (int s = 0; s < depth; ++s) {
        const int c = plan.cells[s];
        set(c);
        if (symmetric) set((c / n) * n + (n - 1 - c % n));
    }
    prm->donate = 1;
    return DLS_OK;
}

int launch(int n, bool vs, const Params &prm, cudaStream_t stream) {
    KernelFn fn = pick_kernel(n, vs);
    if (!fn) { dls::set_error("no kernel for this order"); return DLS_E_ARG; }
    const size_t smem = (size_t)(((prm.L + 2 + 3) & ~3) + (prm.L + 2) * kBlock) * sizeof(uint32_t);
    cudaError_t e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return cuda_fail(e, "cudaDeviceGetAttribute");
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)fn, kBlock, smem)) != cudaSuccess)
        return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (per_sm < 1) { dls::set_error("kernel does not fit on an SM"); return DLS_E_CUDA; }
    long long want_blocks = (long long)sms * per_sm;
    const long long need = (prm.n_prefix + kBlock - 1) / kBlock;  // no more CTAs than work
    if (need < want_blocks) want_blocks = need > 0 ? need : 1;
    fn<<<(unsigned)want_blocks, kBlock, smem, stream>>>(prm);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "kernel launch");
    return DLS_OK;
}

int have_device() {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        dls::set_error("no CUDA device: the B200 path is the only path (no CPU fallback)");
        return DLS_E_NODEVICE;
    }
    return DLS_OK;
}

bool is_device_ptr(const void *ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" int dls_kernel_launches(void) { return 1; }

extern "C" const char *dls_version(void) { return "dls_b200 0.1.0 sm_100a"; }

extern "C" int dls_count_async(int n, int symmetric, int fixed_first_row, int depth,
                               const uint8_t *d_prefixes, int64_t n_prefix, uint64_t *d_counts,
                               uint64_t *d_stats, void *stream) {
    int rc = have_device();
    if (rc) return rc;
    if (n_prefix < 0 || (n_prefix > 0 && !d_prefixes) || !d_stats) {
        dls::set_error("dls_count_async: bad pointers / sizes");
        return DLS_E_ARG;
    }
    Params prm;
    if ((rc = prepare(n, symmetric, fixed_first_row, depth, &prm))) return rc;
    prm.prefixes = d_prefixes;
    prm.n_prefix = n_prefix;
    prm.counts = (u64 *)d_counts;
    prm.stats = (u64 *)d_stats;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d_stats, 0, DLS_STATS_WORDS * sizeof(u64), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(stats)");
    if (d_counts && n_prefix) {
        e = cudaMemsetAsync(d_counts, 0, (size_t)n_prefix * sizeof(u64), s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counts)");
    }
    if (n_prefix == 0) return DLS_OK;
    return launch(n, symmetric, prm, s);
}

namespace {

// Records below which dls_count refines its input (about 8 records per lane of a
// full B200 launch: 148 SMs x 1024 lanes).
constexpr int64_t kRefineTarget = 1200000;
constexpr int kMinSearchLevels = 8;

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
};

}  // namespace

extern "C" int dls_count(int n, int symmetric, int fixed_first_row, int depth,
                         const uint8_t *prefix_buf, int64_t n_prefix, uint64_t *out_counts,
                         uint64_t *out_total, uint64_t *out_nodes, void *stream) {
    int rc = have_device();
    if (rc) return rc;
    if (n_prefix < 0 || (n_prefix > 0 && !prefix_buf)) {
        dls::set_error("dls_count: bad pointers / sizes");
        return DLS_E_ARG;
    }
    dls::Plan plan;
    Params prm;
    if ((rc = prepare(n, symmetric, fixed_first_row, depth, &prm))) return rc;
    dls::make_plan(n, symmetric, fixed_first_row, &plan);
    cudaStream_t s = (cudaStream_t)stream;
    const int nn = n * n;
    const int steps = (int)plan.cells.size();
    cudaError_t e;

    // ---- few, large workunits: cut them deeper on the host (P:481 decomposition
    // applied again below each record) so that every lane of the grid has work.
    const bool in_dev = n_prefix > 0 && is_device_ptr(prefix_buf);
    std::vector<uint8_t> h_in, h_sub;
    std::vector<uint32_t> h_parent;
    const uint8_t *src = prefix_buf;
    int64_t n_rec = n_prefix;
    int depth_run = depth;
    int64_t extra_nodes = 0;
    bool bad_prefix = false;
    if (n_prefix > 0 && n_prefix < kRefineTarget / 8 && depth + 1 <= steps - kMinSearchLevels) {
        if (in_dev) {
            h_in.resize((size_t)n_prefix * nn);
            if ((e = cudaMemcpyAsync(h_in.data(), prefix_buf, h_in.size(), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
                (e = cudaStreamSynchronize(s)) != cudaSuccess)
                return cuda_fail(e, "cudaMemcpy(prefix D2H)");
            src = h_in.data();
        }
        for (int64_t p = 0; p < n_prefix; ++p)
            if (!dls::valid_record(plan, depth, src + p * nn)) bad_prefix = true;
        int d1 = depth;
        int64_t cnt = n_prefix;
        while (cnt < kRefineTarget && d1 + 1 <= steps - kMinSearchLevels) {
            ++d1;
            cnt = dls::refine(plan, depth, d1, src, n_prefix, nullptr, nullptr, 0, nullptr);
        }
        h_sub.resize((size_t)cnt * nn + 1);
        h_parent.resize((size_t)cnt + 1);
        dls::refine(plan, depth, d1, src, n_prefix, h_sub.data(), h_parent.data(), cnt, &extra_nodes);
        if ((rc = prepare(n, symmetric, fixed_first_row, d1, &prm))) return rc;
        src = h_sub.data();
        n_rec = cnt;
        depth_run = d1;
    }
    const bool refined = depth_run != depth;

    DevBuf b_pre, b_cnt, b_par, b_stats;
    const uint8_t *d_pre = src;
    if (n_rec > 0 && (refined || !in_dev)) {
        if ((e = cudaMalloc(&b_pre.p, (size_t)n_rec * nn)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        if ((e = cudaMemcpyAsync(b_pre.p, src, (size_t)n_rec * nn, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpyAsync(H2D)");
        d_pre = (const uint8_t *)b_pre.p;
    }
    u64 *d_counts = (u64 *)out_counts;
    const bool counts_host = out_counts && n_prefix > 0 && !is_device_ptr(out_counts);
    if (counts_host) {
        if ((e = cudaMalloc(&b_cnt.p, (size_t)n_prefix * sizeof(u64))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        d_counts = (u64 *)b_cnt.p;
    }
    if (refined) {
        if ((e = cudaMalloc(&b_par.p, (size_t)n_rec * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        if ((e = cudaMemcpyAsync(b_par.p, h_parent.data(), (size_t)n_rec * sizeof(uint32_t), cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    }
    if ((e = cudaMalloc(&b_stats.p, DLS_STATS_WORDS * sizeof(u64))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    u64 *d_stats = (u64 *)b_stats.p;
    if ((e = cudaMemsetAsync(d_stats, 0, DLS_STATS_WORDS * sizeof(u64), s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync(stats)");
    if (d_counts && n_prefix > 0 &&
        (e = cudaMemsetAsync(d_counts, 0, (size_t)n_prefix * sizeof(u64), s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync(counts)");
    if (n_rec > 0) {
        prm.prefixes = d_pre;
        prm.n_prefix = n_rec;
        prm.counts = d_counts;
        prm.parent = refined ? (const uint32_t *)b_par.p : nullptr;
        prm.stats = d_stats;
        if ((rc = launch(n, symmetric, prm, s))) { cudaStreamSynchronize(s); return rc; }
    }
    u64 stats[DLS_STATS_WORDS];
    if ((e = cudaMemcpyAsync(stats, d_stats, sizeof(stats), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync(stats)");
    if (counts_host &&
        (e = cudaMemcpyAsync(out_counts, d_counts, (size_t)n_prefix * sizeof(u64), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    if (out_total) *out_total = stats[0];
    if (out_nodes) *out_nodes = stats[1] + (prm.L > 0 ? stats[0] : 0) + (u64)extra_nodes;
    if (stats[2] || bad_prefix) {
        dls::set_error("dls_count: some prefix record is not a consistent depth-d prefix");
        return DLS_E_PREFIX;
    }
    return DLS_OK;
}
