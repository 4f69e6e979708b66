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
//    step, chosen branch-free among  descend  (take the lowest candidate of the
//    current cell),  advance  (unmark the value of the previous cell and
//    mark its next candidate in ONE toggle: Alg. 4's "L &= L-1" then "LS = L & -L")
//    and  backtrack; all busy lanes of a warp execute the same instructions;
//  * per-level candidate sets (Alg. 4's L[i][j]) live in a per-lane stack in
//    shared memory, u32 (u16 for N = 9, 10 DLS) per level, layout [level][lane]
//    (bank-conflict free);
//    the lowest set bit of a stacked L is the value assigned at that level;
//  * Rows/Columns occupancy sets are bit fields in registers.  N <= 8: byte fields
//    in 32-bit words -- a cell's candidates are two PRMT byte-selects and one LOP3,
//    marks/unmarks are IMADs with per-cell power-of-two multipliers (FMA pipe,
//    leaving the ALU pipe to the control flow).  VS N = 10: fields in two words
//    per set, funnel-shift reads.  DLS N = 9, 10: three 9/10-bit fields per
//    word, IMAD toggles, word-select + funnel-shift reads (layouts 3, 4; the
//    64-bit-word layout 2 is kept as their A/B baseline).  Per-transition
//    geometry comes pre-decoded from a table;
//  * a global atomic work queue hands prefixes to lanes (one atomic per warp
//    refill); once it is drained, idle lanes receive the untried siblings of the
//    shallowest open level of a busy lane of their warp (warp-vote donation);
//  * counts: 32-bit per burst -> 64-bit per lane -> atomicAdd per prefix
//    (optional) and one 64-bit atomicAdd per block for the total.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "internal.h"

namespace {

typedef unsigned long long u64;

constexpr int kMaxLevels = 100;     // n*n for n = 10
#ifndef DLS_BURST
#define DLS_BURST 256
#endif
constexpr int kBurst = DLS_BURST;   // DFS steps between warp scheduling points
// Shared-memory wavefronts bound the byte-layout kernel (ncu: LSU data pipe at
// 97-98% of peak).  DLS_ONE_STORE=1 (default): the push (descend, slot lvl+1)
// and the rewrite (advance, slot lvl) of a stack slot are one predicated store
// at slot nl -- the slot both write and the one the next step loads; 0 = two
// predicated stores (A/B baseline).
// DLS_LAYOUT9 / DLS_LAYOUT10: mask layout of DLS N = 9 / 10 (2 = 64-bit words +
//   XOR toggles; 3 / 4 = three 9- / 10-bit fields per 32-bit word + IMAD toggles)
#ifndef DLS_LAYOUT9
#define DLS_LAYOUT9 3
#endif
#ifndef DLS_LAYOUT10
#define DLS_LAYOUT10 4
#endif
#ifndef DLS_ONE_STORE
#define DLS_ONE_STORE 1
#endif
// DLS_UNIFIED=1 (default): byte layout (N <= 8), 1024 lanes: a transition block
// and a stack slot are both 1024 bytes, so ONE register -- the shared address of
// the lane's table entry of the current level -- stands for the level; table and
// stack addresses are that register plus per-lane constants (4 level
// instructions per step instead of 7).  0 = the generic step (A/B baseline).
#ifndef DLS_UNIFIED
#define DLS_UNIFIED 1
#endif
// DLS_READ8=1: the byte layout's 8-byte read entries at an 8-byte lane stride (2
// shared-memory wavefronts instead of 4).  DLS_FMA_ADDS=1: the level / address
// additions of the unified step are written as multiply-adds with a factor the
// compiler cannot see (Params::one = 1), so they issue on the FMA pipe instead
// of the half-rate ALU pipe, which binds the step (profiles/r2_ab_step.log).
#ifndef DLS_READ8
#define DLS_READ8 0
#endif
#ifndef DLS_FMA_ADDS
#define DLS_FMA_ADDS 0
#endif
// DLS_STEP_V2=1: the unified step selects the L set it works on first (one
// select, one lowest-bit isolation instead of two) -- fewer ALU-pipe instructions
#ifndef DLS_STEP_V2
#define DLS_STEP_V2 1
#endif
// steps between two looks at the event stacks in the kernels with 8-byte events
// (their stacks are twice as deep)
#ifndef DLS_GROUP8
#define DLS_GROUP8 8
#endif
// kernels with 8-byte events: 1 = closure rounds start when a stack nears its
// depth (one vote per look), 0 = when enough lanes hold an event (a reduction)
#ifndef DLS_ROUNDS_ON_FULL
#define DLS_ROUNDS_ON_FULL 1
#endif

// A closure round (every lane evaluates its newest event) starts once this many
// lanes of the warp hold one (A/B: profiles/r2_ab_close_min.log)
constexpr int kCloseMinLanes = 24;
constexpr int kMinDonateDepth = 6;  // do not donate subtrees shallower than this (and < L/3)
constexpr unsigned kFull = 0xFFFFFFFFu;

// Internal invariants, compiled in only with -DDLS_CHECKS (the checked build,
// libdls_b200_checked.so): a violated one sets bit 8 + k of the error word
// stats[2] (bit 0 stays the prefix-error flag) and the host call fails with
// DLS_E_CUDA.  The product build compiles them out.
#ifdef DLS_CHECKS
#define DLS_CHECK(cond, k) do { if (!(cond)) atomicOr(p.stats + 2, 1ull << (8 + (k))); } while (0)
#else
#define DLS_CHECK(cond, k) do { } while (0)
#endif
enum CheckBits {
    kChkStep = 0,       // DFS step: slot / table indices inside levels -1 .. L+1
    kChkAdopt = 1,      // adopted workunit: pid < n_prefix, split in 0 .. L
    kChkPoolPut = 2,    // pool producer: slot not still owned by an unread ticket
    kChkPoolGet = 3,    // pool consumer: pid / split of a claimed slot in range
    kChkWarpGive = 4,   // intra-warp donation: the source lane really donates
    kChkExit = 5,       // kernel exit: every lane idle, levels -1 / 0 untouched
    kChkEmit = 6,       // emitted square: pid in range
};
// Device-wide donation pool (global memory, one per launch): control words
// [0] active warps, [1] waiting warps, [2] head (claimed), [3] tail (reserved),
// [4] warps registered (exit is allowed only once all warps of the grid are),
// [5] slots released (read completely; producers bound tail - released so a
//     claimed slot is never overwritten before its reader is done),
// then kPoolSlots slots of kSlotWords: w0 = ticket+1 once written, w1 = pid,
// w2 = ticket+1 once read (a producer of the next lap waits for it),
// w3 = split level | untried siblings << 16, w4.. = the values (bit indices) of
// levels 1..split-1, 4 bits each.
constexpr uint32_t kPoolSlots = 16384;
constexpr uint32_t kPoolLimit = 8192;   // producers stop while this many are pending
constexpr int kSlotWords = 32;
constexpr int kPoolHeader = 32;
constexpr size_t kPoolBytes = (size_t)(kPoolHeader + kPoolSlots * kSlotWords) * 4;

// One transition t (t = -1 .. L): "toggle a value at cell(t), then read the
// candidates of cell(t+1)".  Eight words; the meaning depends on the mask layout.
struct Tab {
    uint32_t w[8];
};

struct Params {
    const uint8_t *prefixes;
    long long n_prefix;
    u64 *counts;             // per-prefix counts (may be null)
    const uint32_t *parent;  // record -> output slot (null = identity; set by refinement)
    u64 *stats;              // DLS_STATS_WORDS words, see dls_b200.h
    uint32_t *pool;          // device-wide donation pool (kPoolBytes, zeroed)
    u64 pat[2];              // cells assigned in a prefix, bit i*n+j
    int L;                   // number of searched levels (plan cells after the prefix)
    int donate;              // enable warp-level subtree donation
    int min_donate;          // smallest donated subtree (levels below the split)
    uint32_t total_warps;    // warps of the grid (exit once all registered)
    uint8_t *emit;           // emit kernels: complete squares, n*n bytes each
    long long emit_cap;      //               capacity (records)
    // two-row closure: the search stops at level L,
    // where only rows r1, r2 still have empty cells, all in the same columns and
    // off both diagonals; the completions of such a state are counted in closed
    // form from the column sets and row r1 (close_count)
    int close;               // 1: level L+1 is a closure event (CLOSE kernels)
    uint32_t cl_open;        // tracked columns with empty cells in rows r1, r2
    int cl_E;                // popc(cl_open)
    int cl_rword;            // mask-layout word holding row r1's field
    // layouts 3, 4: rows cl_swap_a and cl_swap_b trade their fields (-1: none), so
    // that row r1 always sits in word R[2] and the event store needs no select
    int cl_swap_a, cl_swap_b;
    int cl_rshift;           // bit offset of row r1's field in that word
    uint32_t cl_sel[10];     // field selectors of the columns of J (padded)
    int cl_min;              // lanes of a warp holding an event that start an evaluation round
    int cl_cq;               // event slots per lane (set by launch from the shared memory left)
    uint32_t one;            // 1 (see DLS_FMA_ADDS)
    // forced cells just before the two-row level, assigned inside the closure
    // (their value is the one candidate their complete-but-one row or column
    // leaves): read entry (words 4..7) and toggle entry (words 0..7) of each
    int cl_nf;
    Tab cl_fread[2], cl_ftog[2];
    // lookahead (Section 2.4.2; LOOK kernels, DLS N = 9): after the
    // toggle of transition t also read the candidates of a watched cell; none
    // left -> the branch is cut.  look_sel[t + 1] = its row / column selectors
    // (transitions without a watched cell watch cell(t+1) itself: a no-op)
    int look;
    uint32_t look_sel[kMaxLevels + 2][2];
    uint8_t level_cell[kMaxLevels + 2];   // cell (i*n+j) of level l = 1..L
    Tab tab[kMaxLevels + 2]; // tab[t + 1], t = -1 .. L
};

// ---------------------------------------------------------------- mask layouts

// Row sets: for DLS the N value bits of a row; for vertical symmetry N/2 "pair"
// bits (a row always holds v and N-1-v together), and only the N/2 left columns
// are tracked (column N-1-j is the mirror of column j).
template <int N, bool VS>
struct Geo {
    static constexpr int H = N / 2;
    static constexpr int NC = VS ? H : N;                      // tracked columns
    static constexpr uint32_t ALLN = (1u << N) - 1u;
    static constexpr uint32_t HMASK = (1u << H) - 1u;
    static constexpr int RF = VS ? (H > 0 ? H : 1) : N;        // row field width (bits)
    static constexpr int CF = N;                               // column field width
    // word-field layout: fields never straddle a 32-bit word, 2 words per unit
    static constexpr int RPW32 = 32 / RF;
    static constexpr int CPW32 = 32 / CF;
    static constexpr bool FITS2 = (N + RPW32 - 1) / RPW32 <= 2 && (NC + CPW32 - 1) / CPW32 <= 2;
    // 0: byte fields + PRMT (N <= 8); 1: word fields + funnel shift (e.g. VS N=10);
    // 2: 64-bit words + funnel shifts (A/B baseline); 3 / 4: three 9 / 10-bit
    // fields per word + IMAD toggles (DLS N = 9 / 10)
    static constexpr int LAYOUT = N <= 8 ? 0
                                : FITS2 ? 1
                                : (N == 9 && !VS && DLS_LAYOUT9 == 3) ? 3
                                : (N == 10 && !VS && DLS_LAYOUT10 == 4) ? 4 : 2;
    static constexpr bool BYTES = LAYOUT == 0;
    static constexpr int RPW = 64 / RF;                        // layout 2
    static constexpr int CPW = 64 / CF;
    static constexpr int WR = (N + RPW - 1) / RPW;
    static constexpr int WC = (NC + CPW - 1) / CPW;
    // value v -> bit position inside the kernel.  DLS: v.  VS: the mirror of
    // position p is p +- H, so a row's pair mask expands with one IMAD.
    __host__ __device__ static constexpr int pos(int v) {
        return !VS ? v : (v < H ? v : H + (N - 1 - v));
    }
    // value bit -> row-field bit
    __device__ __forceinline__ static uint32_t rowbit(uint32_t b) {
        return VS ? ((b | (b >> H)) & HMASK) : b;
    }
    __device__ __forceinline__ static uint32_t expand_row(uint32_t r) {
        return VS ? (r & HMASK) * ((1u << H) + 1u) : r;
    }
};

template <int N, bool VS, int LAYOUT = Geo<N, VS>::LAYOUT>
struct Masks;

// N <= 8: row r is byte r&3 of R[r>>2], column c is byte c&3 of C[c>>2].
// Tab: w0..w3 = multipliers of cell(t)'s row/col byte in R0,R1,C0,C1
//      (1 << 8*(r&3) in the word holding the field, 0 in the other);
//      w4, w5 = PRMT selectors (row, col byte index 0..7) of cell(t+1).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

template <int N, bool VS>
struct Masks<N, VS, 0> {
    typedef Geo<N, VS> G;
    typedef uint2 CT;
    uint32_t R0, R1, C0, C1;

    __device__ __forceinline__ void clear() { R0 = R1 = C0 = C1 = 0; }
    __device__ __forceinline__ void set_row(int r, uint32_t m) { if (r < 4) R0 |= m << (8 * r); else R1 |= m << (8 * (r - 4)); }
    __device__ __forceinline__ void set_col(int c, uint32_t m) { if (c < 4) C0 |= m << (8 * c); else C1 |= m << (8 * (c - 4)); }
    // fields change by +bnew -bold (bnew absent, bold present: no carries between fields)
    __device__ __forceinline__ void toggle(const uint4 &f, uint32_t bnew, uint32_t bold) {
        const uint32_t dc = bnew - bold;
        const uint32_t dr = VS ? G::rowbit(bnew) - G::rowbit(bold) : dc;
        toggle_d(f, dr, dc);
    }
    __device__ __forceinline__ void toggle_d(const uint4 &f, uint32_t dr, uint32_t dc) {
        R0 += dr * f.x;      // IMAD: mark/unmark on the FMA pipe
        R1 += dr * f.y;
        C0 += dc * f.z;
        C1 += dc * f.w;
    }
    __device__ __forceinline__ uint32_t cand(const uint2 &c) const {
        const uint32_t r = G::expand_row(prmt(R0, R1, c.x));
        const uint32_t k = prmt(C0, C1, c.y);
        return G::ALLN & ~(r | k);                               // AllN ^ (Rows | Columns)
    }
};

// Word fields (e.g. vertical symmetry, N = 10): row r is field r % RPW32 of
// R[r / RPW32] (RF bits each), column c field c % CPW32 of C[c / CPW32]; no field
// straddles a word, so toggles are IMADs as in the byte layout, and a field is read
// with one 64-bit funnel shift of the word pair.
// Tab: w0..w3 = multipliers (1 << field offset, in the word holding the field);
//      w4, w5 = bit offsets (0..63) of cell(t+1)'s row/col field in the pair.
template <int N, bool VS>
struct Masks<N, VS, 1> {
    typedef Geo<N, VS> G;
    typedef uint4 CT;
    uint32_t R0, R1, C0, C1;

    __device__ __forceinline__ void clear() { R0 = R1 = C0 = C1 = 0; }
    __device__ __forceinline__ void set_row(int r, uint32_t m) {
        const int o = (r % G::RPW32) * G::RF;
        if (r / G::RPW32 == 0) R0 |= m << o; else R1 |= m << o;
    }
    __device__ __forceinline__ void set_col(int c, uint32_t m) {
        const int o = (c % G::CPW32) * G::CF;
        if (c / G::CPW32 == 0) C0 |= m << o; else C1 |= m << o;
    }
    __device__ __forceinline__ void toggle(const uint4 &f, uint32_t bnew, uint32_t bold) {
        const uint32_t dc = bnew - bold;
        const uint32_t dr = VS ? G::rowbit(bnew) - G::rowbit(bold) : dc;
        R0 += dr * f.x;
        R1 += dr * f.y;
        C0 += dc * f.z;
        C1 += dc * f.w;
    }
    __device__ __forceinline__ uint32_t cand(const uint4 &c) const {
        const uint32_t r = G::expand_row((uint32_t)((((u64)R1 << 32) | R0) >> c.x));
        const uint32_t k = (uint32_t)((((u64)C1 << 32) | C0) >> c.y);
        return G::ALLN & ~(r | k);
    }
};

// 64-bit words (the A/B baseline of DLS N = 9, 10): row/column fields packed in
// W words, moved by funnel shifts.  Tab: w0..w3 = row shift, row word, col shift, col word of
// cell(t); w4..w7 = the same of cell(t+1).
template <int N, bool VS>
struct Masks<N, VS, 2> {
    typedef Geo<N, VS> G;
    u64 R[G::WR];
    u64 C[G::WC];

    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int w = 0; w < G::WR; ++w) R[w] = 0;
#pragma unroll
        for (int w = 0; w < G::WC; ++w) C[w] = 0;
    }
    __device__ __forceinline__ void set_row(int r, uint32_t m) { R[r / G::RPW] |= (u64)m << ((r % G::RPW) * G::RF); }
    __device__ __forceinline__ void set_col(int c, uint32_t m) { C[c / G::CPW] |= (u64)m << ((c % G::CPW) * G::CF); }
    template <int W>
    __device__ __forceinline__ static void flip(u64 (&a)[W], uint32_t sh, uint32_t wd, uint32_t bits) {
        const u64 t = (u64)bits << sh;
        if (W == 1) {
            a[0] ^= t;
        } else {
            a[0] ^= wd ? 0ull : t;
            a[W - 1] ^= wd ? t : 0ull;
        }
    }
    template <int W>
    __device__ __forceinline__ static uint32_t field(const u64 (&a)[W], uint32_t sh, uint32_t wd) {
        u64 w = a[0];
        if (W == 2) w = wd ? a[W - 1] : a[0];
        return (uint32_t)(w >> sh);
    }
    __device__ __forceinline__ void toggle(const uint4 &f, uint32_t bnew, uint32_t bold) {
        const uint32_t xc = bnew ^ bold;
        const uint32_t xr = VS ? (G::rowbit(bnew) ^ G::rowbit(bold)) : xc;
        flip<G::WR>(R, f.x, f.y, xr);
        flip<G::WC>(C, f.z, f.w, xc);
    }
    __device__ __forceinline__ uint32_t cand(const uint4 &c) const {
        const uint32_t r = G::expand_row(field<G::WR>(R, c.x, c.y));
        const uint32_t k = field<G::WC>(C, c.z, c.w);
        return G::ALLN & ~(r | k);
    }

    typedef uint4 CT;
};

// DLS N = 9: three 9-bit fields per 32-bit word, R[3] rows and C[3] columns, so
// a toggle is six IMADs with per-word multipliers (0 for the words without the
// field; signed deltas never carry between fields, as in the byte layout).
// Tab: w0..w2 = row-word multipliers of cell(t), w3..w5 = column-word
//      multipliers, w6 / w7 = row / column selector of cell(t+1): bit offset in
//      the word (0, 9, 18) | word index << 5.
template <int N, bool VS>
struct Masks<N, VS, 3> {
    typedef Geo<N, VS> G;
    typedef uint4 CT;
    static constexpr int FPW = 32 / N;
    static_assert(!VS && FPW == 3 && (N + FPW - 1) / FPW == 3, "layout 3 is DLS N = 9");
    uint32_t R[3], C[3];

    __device__ __forceinline__ void clear() { R[0] = R[1] = R[2] = C[0] = C[1] = C[2] = 0; }
    __device__ __forceinline__ void set_row(int r, uint32_t m) { R[r / FPW] |= m << ((r % FPW) * N); }
    __device__ __forceinline__ void set_col(int c, uint32_t m) { C[c / FPW] |= m << ((c % FPW) * N); }
    __device__ __forceinline__ void toggle_d(const uint4 &f, const uint4 &g, uint32_t d) {
        R[0] += d * f.x;     // IMAD: mark/unmark on the FMA pipe
        R[1] += d * f.y;
        R[2] += d * f.z;
        C[0] += d * f.w;
        C[1] += d * g.x;
        C[2] += d * g.y;
    }
    __device__ __forceinline__ void toggle(const uint4 &f, const uint4 &g, uint32_t bnew, uint32_t bold) {
        toggle_d(f, g, bnew - bold);
    }
    // rows a and b trade their fields (once per adopted record)
    __device__ __forceinline__ void swap_rows(int a, int b) {
        const int sa = (a % FPW) * N, sb = (b % FPW) * N;
        const uint32_t wa = a / FPW == 0 ? R[0] : (a / FPW == 1 ? R[1] : R[2]);
        const uint32_t wb = b / FPW == 0 ? R[0] : (b / FPW == 1 ? R[1] : R[2]);
        const uint32_t x = ((wa >> sa) ^ (wb >> sb)) & G::ALLN;
#pragma unroll
        for (int w = 0; w < 3; ++w) R[w] ^= (a / FPW == w ? x << sa : 0u) ^ (b / FPW == w ? x << sb : 0u);
    }
    __device__ __forceinline__ static uint32_t pick(const uint32_t (&a)[3], uint32_t sel) {
        const uint32_t w = (sel & 64u) ? a[2] : ((sel & 32u) ? a[1] : a[0]);
        return __funnelshift_r(w, 0u, sel);          // shift by sel & 31
    }
    __device__ __forceinline__ uint32_t cand(const uint4 &c) const {
        return G::ALLN & ~(pick(R, c.z) | pick(C, c.w));
    }
};

// DLS N = 10: three 10-bit fields per 32-bit word.  Rows 1..9 in R[3] (row r at
// word (r-1)/3), columns 0..8 in C[3], and X = column 9 (offset 0) | row 0
// (offset 10): seven IMAD toggles (a cell of row 0 or column 9 has a multiplier
// on X; cell (0, 9) has 1 + 2^10 there).  Tab: w0..w2 = R multipliers, w3..w5 =
// C multipliers, w6 = X multiplier, w7 = row selector | column selector << 16
// (selector = bit offset | word << 5, word 3 = X).
template <int N, bool VS>
struct Masks<N, VS, 4> {
    typedef Geo<N, VS> G;
    typedef uint4 CT;
    static_assert(!VS && N == 10, "layout 4 is DLS N = 10");
    uint32_t R[3], C[3], X;

    __device__ __forceinline__ void clear() { R[0] = R[1] = R[2] = C[0] = C[1] = C[2] = X = 0; }
    __device__ __forceinline__ void set_row(int r, uint32_t m) {
        if (r == 0) X |= m << N;
        else R[(r - 1) / 3] |= m << (((r - 1) % 3) * N);
    }
    __device__ __forceinline__ void set_col(int c, uint32_t m) {
        if (c == N - 1) X |= m;
        else C[c / 3] |= m << ((c % 3) * N);
    }
    __device__ __forceinline__ void toggle_d(const uint4 &f, const uint4 &g, uint32_t d) {
        R[0] += d * f.x;     // IMAD: mark/unmark on the FMA pipe
        R[1] += d * f.y;
        R[2] += d * f.z;
        C[0] += d * f.w;
        C[1] += d * g.x;
        C[2] += d * g.y;
        X += d * g.z;
    }
    __device__ __forceinline__ void toggle(const uint4 &f, const uint4 &g, uint32_t bnew, uint32_t bold) {
        toggle_d(f, g, bnew - bold);
    }
    // rows a, b >= 1 trade their fields (once per adopted record)
    __device__ __forceinline__ void swap_rows(int a, int b) {
        const int ia = a - 1, ib = b - 1;
        const int sa = (ia % 3) * N, sb = (ib % 3) * N;
        const uint32_t wa = ia / 3 == 0 ? R[0] : (ia / 3 == 1 ? R[1] : R[2]);
        const uint32_t wb = ib / 3 == 0 ? R[0] : (ib / 3 == 1 ? R[1] : R[2]);
        const uint32_t x = ((wa >> sa) ^ (wb >> sb)) & G::ALLN;
#pragma unroll
        for (int w = 0; w < 3; ++w) R[w] ^= (ia / 3 == w ? x << sa : 0u) ^ (ib / 3 == w ? x << sb : 0u);
    }
    __device__ __forceinline__ static uint32_t pick(const uint32_t (&a)[3], uint32_t x, uint32_t sel) {
        const uint32_t w = (sel & 64u) ? ((sel & 32u) ? x : a[2]) : ((sel & 32u) ? a[1] : a[0]);
        return __funnelshift_r(w, 0u, sel);          // shift by sel & 31
    }
    __device__ __forceinline__ uint32_t cand(const uint4 &c) const {
        return G::ALLN & ~(pick(R, X, c.w) | pick(C, X, c.w >> 16));
    }
};

// ---------------------------------------------------------------- two-row closure
//
// At the closure level every row except r1, r2 is complete, the empty cells of
// r1 and r2 lie in the same columns J and on neither diagonal.  Each column j in
// J then misses exactly two values e_j, and a value v is missing from
// m1(v) + m2(v) columns of J (m_r(v) = 1 if row r misses v; counting argument,
// DESIGN.md "Tail closure").  A completion is a choice p_j in e_j for row r1
// (row r2 takes the other value) such that row r1 receives each of its missing
// values once; with the degrees above this is exactly the GF(2) condition
//     XOR_j p_j = M1   <=>   XOR_{j: x_j = 1} e_j = t,
//     t = M1 ^ XOR_j low(e_j)      (x_j = 1: row r1 takes the higher value),
// whose number of solutions is 2^(|J| - rank) if t lies in the span of the e_j
// and 0 otherwise.  Row r2 is then complete and valid by the same counting.
// Vertical symmetry: the same over the N/2 value pairs {v, N-1-v} of the left
// columns, e_j = fold(missing positions) (a column missing both values of one
// pair gives e_j = 0: two completions that differ in that column).
//
// A closure event stores the part of the state it needs (the column words and
// the words holding row r1) on its lane's event stack in shared memory; once
// enough lanes of the warp hold an event, every lane evaluates its newest one
// (Close::eval) -- the same instructions in all lanes.  The host
// lists the columns of J as layout-specific field selectors (cl_sel), padded to
// EM entries with a complete column (its missing set is empty).
template <int N, bool VS, int LAYOUT = Geo<N, VS>::LAYOUT>
struct Close;

template <int N, bool VS>
struct CloseBase {
    typedef Geo<N, VS> G;
    static constexpr uint32_t RMASK = VS ? G::HMASK : G::ALLN;
    // |J| <= EM: rows r1 != r2 close >= 2 diagonal columns (DLS) / >= 1 left one (VS)
    static constexpr int EM = VS ? (G::H > 1 ? G::H - 1 : 1) : (N > 2 ? N - 2 : 1);
    __device__ __forceinline__ static uint32_t fold(uint32_t m) { return VS ? (m ^ (m >> G::H)) & G::HMASK : m; }
    // f[k]: field of the k-th column of J (occupied values / positions)
    __device__ __forceinline__ static uint32_t count(const uint32_t (&f)[EM], uint32_t rowf, const Params &p) {
        uint32_t e[EM];
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < EM; ++k) {
            const uint32_t m = G::ALLN & ~f[k];        // the two values column k misses
            x ^= m & (0u - m);                         // XOR_j low(e_j)
            e[k] = fold(m);
        }
        uint32_t t = fold(x) ^ (RMASK & ~rowf);        // M1 ^ XOR_j low(e_j)
        int rank = 0;
#pragma unroll
        for (int k = 0; k < EM; ++k) {                 // Gaussian elimination over GF(2)
            const uint32_t ek = e[k];
            const uint32_t piv = ek & (0u - ek);
            rank += ek != 0u;
#pragma unroll
            for (int j = k + 1; j < EM; ++j)
                if (e[j] & piv) e[j] ^= ek;
            if (t & piv) t ^= ek;
        }
        return t ? 0u : 1u << (p.cl_E - rank);
    }
};

// byte layout: queue entry {C0, C1, R0, R1}; column selector = byte index
template <int N, bool VS>
struct Close<N, VS, 0> : CloseBase<N, VS> {
    typedef CloseBase<N, VS> B;
    static constexpr int EW = 4;   // words per queue entry
    __device__ __forceinline__ static uint4 pack(const Masks<N, VS> &st, uint32_t) {
        return make_uint4(st.C0, st.C1, st.R0, st.R1);
    }
    __device__ __forceinline__ static uint32_t eval(const uint32_t *src, const Params &p, uint32_t rsel) {
        uint4 w = *reinterpret_cast<const uint4 *>(src);
        bool ok = true;
        if (p.cl_nf) {
            Masks<N, VS> m;
            m.C0 = w.x; m.C1 = w.y; m.R0 = w.z; m.R1 = w.w;
#pragma unroll
            for (int k = 0; k < 2; ++k)
                if (k < p.cl_nf) {
                    const uint32_t v = m.cand(make_uint2(p.cl_fread[k].w[4], p.cl_fread[k].w[5]));
                    ok &= v != 0u;
                    m.toggle(make_uint4(p.cl_ftog[k].w[0], p.cl_ftog[k].w[1], p.cl_ftog[k].w[2], p.cl_ftog[k].w[3]), v, 0u);
                }
            w = make_uint4(m.C0, m.C1, m.R0, m.R1);
        }
        const uint32_t c = eval_cols(w.x, w.y, ((rsel ? w.w : w.z) >> p.cl_rshift) & 0xFFu, p);
        return ok ? c : 0u;
    }
    // the count from the column words and row r1's field (8-byte events, CROW
    // kernels: row r1 has no searched cell, its field is a per-workunit constant)
    __device__ __forceinline__ static uint32_t eval_cols(uint32_t c0, uint32_t c1, uint32_t rowf, const Params &p) {
        uint32_t f[B::EM];
#pragma unroll
        for (int k = 0; k < B::EM; ++k) f[k] = prmt(c0, c1, p.cl_sel[k]) & 0xFFu;
        return B::count(f, rowf, p);
    }
};

// word fields (VS N = 10): entry {C0, C1, R0, R1}; selector = bit offset of the
// field in the 64-bit pair C1:C0
template <int N, bool VS>
struct Close<N, VS, 1> : CloseBase<N, VS> {
    typedef CloseBase<N, VS> B;
    typedef Geo<N, VS> G;
    static constexpr int EW = 4;
    __device__ __forceinline__ static uint4 pack(const Masks<N, VS> &st, uint32_t) {
        return make_uint4(st.C0, st.C1, st.R0, st.R1);
    }
    __device__ __forceinline__ static uint32_t eval(const uint32_t *src, const Params &p, uint32_t rsel) {
        uint4 w = *reinterpret_cast<const uint4 *>(src);
        bool ok = true;
        if (p.cl_nf) {
            Masks<N, VS> m;
            m.C0 = w.x; m.C1 = w.y; m.R0 = w.z; m.R1 = w.w;
#pragma unroll
            for (int k = 0; k < 2; ++k)
                if (k < p.cl_nf) {
                    const Tab &rd = p.cl_fread[k], &tg = p.cl_ftog[k];
                    const uint32_t v = m.cand(make_uint4(rd.w[4], rd.w[5], rd.w[6], rd.w[7]));
                    ok &= v != 0u;
                    m.toggle(make_uint4(tg.w[0], tg.w[1], tg.w[2], tg.w[3]), v, 0u);
                }
            w = make_uint4(m.C0, m.C1, m.R0, m.R1);
        }
        const uint32_t c = eval_cols(w.x, w.y, (rsel ? w.w : w.z) >> p.cl_rshift, p);
        return ok ? c : 0u;
    }
    // the count from the column words and row r1's field (8-byte events, CROW kernels)
    __device__ __forceinline__ static uint32_t eval_cols(uint32_t c0, uint32_t c1, uint32_t rowf, const Params &p) {
        uint32_t f[B::EM];
#pragma unroll
        for (int k = 0; k < B::EM; ++k)
            f[k] = (uint32_t)((((u64)c1 << 32) | c0) >> p.cl_sel[k]) & ((1u << G::CF) - 1u);
        return B::count(f, rowf & ((1u << G::RF) - 1u), p);
    }
};

// DLS N = 9: entry {C0, C1, C2, word of row r1}; selector = bit offset | word
// << 5 (as the read entries of layout 3)
template <int N, bool VS>
struct Close<N, VS, 3> : CloseBase<N, VS> {
    typedef CloseBase<N, VS> B;
    static constexpr int EW = 4;
    // (the host moves row r1 into word R[2]: cl_swap_a / cl_swap_b, cl_rword = 2)
    __device__ __forceinline__ static uint4 pack(const Masks<N, VS> &st, uint32_t) {
        return make_uint4(st.C[0], st.C[1], st.C[2], st.R[2]);
    }
    __device__ __forceinline__ static uint32_t eval(const uint32_t *src, const Params &p, uint32_t rsel) {
        uint4 w = *reinterpret_cast<const uint4 *>(src);
        bool ok = true;
        if (p.cl_nf) {   // the forced cells' rows share row r1's word (host check)
            Masks<N, VS, 3> m;
            m.C[0] = w.x; m.C[1] = w.y; m.C[2] = w.z;
            m.R[0] = rsel == 0 ? w.w : 0u; m.R[1] = rsel == 1 ? w.w : 0u; m.R[2] = rsel == 2 ? w.w : 0u;
#pragma unroll
            for (int k = 0; k < 2; ++k)
                if (k < p.cl_nf) {
                    const Tab &rd = p.cl_fread[k], &tg = p.cl_ftog[k];
                    const uint32_t v = m.cand(make_uint4(rd.w[4], rd.w[5], rd.w[6], rd.w[7]));
                    ok &= v != 0u;
                    m.toggle(make_uint4(tg.w[0], tg.w[1], tg.w[2], tg.w[3]), make_uint4(tg.w[4], tg.w[5], tg.w[6], tg.w[7]),
                             v, 0u);
                }
            w = make_uint4(m.C[0], m.C[1], m.C[2], rsel == 2 ? m.R[2] : (rsel == 1 ? m.R[1] : m.R[0]));
        }
        const uint32_t c[3] = {w.x, w.y, w.z};
        uint32_t f[B::EM];
#pragma unroll
        for (int k = 0; k < B::EM; ++k) f[k] = Masks<N, VS, 3>::pick(c, p.cl_sel[k]) & 0x1FFu;
        const uint32_t cnt = B::count(f, (w.w >> p.cl_rshift) & 0x1FFu, p);
        return ok ? cnt : 0u;
    }
};

// DLS N = 10: entry {C0, C1, C2, X} + the word of row r1 (two stores, 20 of the
// slot's 32 bytes); selector as the read entries of layout 4
template <int N, bool VS>
struct Close<N, VS, 4> : CloseBase<N, VS> {
    typedef CloseBase<N, VS> B;
    static constexpr int EW = 8;
    __device__ __forceinline__ static uint4 pack(const Masks<N, VS> &st, uint32_t) {
        return make_uint4(st.C[0], st.C[1], st.C[2], st.X);
    }
    // (the host moves row r1 into word R[2]: cl_swap_a / cl_swap_b, cl_rword = 2)
    __device__ __forceinline__ static uint32_t pack_row(const Masks<N, VS> &st, uint32_t) { return st.R[2]; }
    __device__ __forceinline__ static uint32_t eval(const uint32_t *src, const Params &p, uint32_t rsel) {
        uint4 w = *reinterpret_cast<const uint4 *>(src);
        uint32_t rw = src[4];
        bool ok = true;
        if (p.cl_nf) {   // the forced cells' rows share row r1's word (host check)
            Masks<N, VS, 4> m;
            m.C[0] = w.x; m.C[1] = w.y; m.C[2] = w.z; m.X = w.w;
            m.R[0] = rsel == 0 ? rw : 0u; m.R[1] = rsel == 1 ? rw : 0u; m.R[2] = rsel == 2 ? rw : 0u;
#pragma unroll
            for (int k = 0; k < 2; ++k)
                if (k < p.cl_nf) {
                    const Tab &rd = p.cl_fread[k], &tg = p.cl_ftog[k];
                    const uint32_t v = m.cand(make_uint4(rd.w[4], rd.w[5], rd.w[6], rd.w[7]));
                    ok &= v != 0u;
                    m.toggle(make_uint4(tg.w[0], tg.w[1], tg.w[2], tg.w[3]), make_uint4(tg.w[4], tg.w[5], tg.w[6], tg.w[7]),
                             v, 0u);
                }
            w = make_uint4(m.C[0], m.C[1], m.C[2], m.X);
            rw = rsel == 3 ? m.X : (rsel == 2 ? m.R[2] : (rsel == 1 ? m.R[1] : m.R[0]));
        }
        const uint32_t c[3] = {w.x, w.y, w.z};
        uint32_t f[B::EM];
#pragma unroll
        for (int k = 0; k < B::EM; ++k) f[k] = Masks<N, VS, 4>::pick(c, w.w, p.cl_sel[k]) & 0x3FFu;
        const uint32_t cnt = B::count(f, (rw >> p.cl_rshift) & 0x3FFu, p);
        return ok ? cnt : 0u;
    }
};

// layout 2 (the 64-bit A/B baseline) has no closure: the host never enables it
template <int N, bool VS>
struct Close<N, VS, 2> : CloseBase<N, VS> {
    static constexpr int EW = 4;
    __device__ __forceinline__ static uint4 pack(const Masks<N, VS> &, uint32_t) { return make_uint4(0, 0, 0, 0); }
    __device__ __forceinline__ static uint32_t pack_row(const Masks<N, VS> &, uint32_t) { return 0u; }
    __device__ __forceinline__ static uint32_t eval(const uint32_t *, const Params &, uint32_t) { return 0u; }
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ u64 globaltimer() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Timeline stamps (ns, %globaltimer) in the pool header, read back by the host
// under DLS_TIMING: first warp start, queue found empty, first CTA exit, last
// CTA exit -- the length of the end-game after the work queue runs dry.
constexpr int kStampStart = 6, kStampQEmpty = 8, kStampFirstExit = 10, kStampLastExit = 12;
__device__ __forceinline__ void stamp_first(uint32_t *pool, int w) {
    atomicCAS(reinterpret_cast<u64 *>(pool + w), 0ull, globaltimer());
}

__host__ __device__ inline bool pat_bit(const u64 *pat, int c) {
    return (pat[c >> 6] >> (c & 63)) & 1ull;
}

// Build the row/column sets of one prefix record and validate it: exactly the
// pattern cells assigned, values < N, no repeated value in a row, column or
// diagonal, and (VS) mirror consistency LS[i][N-1-j] = N-1-LS[i][j].
template <int N, bool VS>
__device__ __forceinline__ bool load_prefix(const uint8_t *__restrict__ rec, const u64 pat0, const u64 pat1,
                                            Masks<N, VS> &st) {
    typedef Geo<N, VS> G;
    const u64 pat[2] = {pat0, pat1};
    uint32_t cm[N];                                 // value bits per column (validation)
    uint32_t sc[VS ? (G::NC > 0 ? G::NC : 1) : 1];  // VS: position bits of the left columns
    uint32_t md = 0, ad = 0;
    bool ok = true;
    st.clear();
#pragma unroll
    for (int j = 0; j < N; ++j) cm[j] = 0;
#pragma unroll
    for (int j = 0; j < (VS ? G::NC : 1); ++j) sc[j] = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        uint32_t rm = 0, sr = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const uint32_t v = __ldg(rec + i * N + j);
            const bool assigned = v != DLS_EMPTY;
            ok &= assigned == pat_bit(pat, i * N + j);
            if (assigned) {
                ok &= v < (uint32_t)N;
                const uint32_t b = 1u << (v & 31u);
                ok &= !(rm & b) && !(cm[j] & b);
                rm |= b;
                cm[j] |= b;
                if (i == j) { ok &= !(md & b); md |= b; }
                if (i + j == N - 1) { ok &= !(ad & b); ad |= b; }
                if (VS) {
                    const uint32_t m = __ldg(rec + i * N + (N - 1 - j));
                    ok &= m == (uint32_t)(N - 1) - v;
                    const uint32_t pb = 1u << (G::pos((int)(v & 15u)) & 31);
                    if (2 * j < N - 1) {
                        sr |= G::rowbit(pb);
                        sc[j < G::NC ? j : 0] |= pb;
                    }
                }
            }
        }
        st.set_row(i, VS ? sr : rm);
    }
#pragma unroll
    for (int j = 0; j < G::NC; ++j) st.set_col(j, VS ? sc[VS ? j : 0] : cm[j]);
    return ok;
}


// Shared memory of one CTA (one CTA per SM, NT lanes):
//   per transition u = t+1 (t = -1 .. L) a block of 32 toggle entries (uint4)
//   followed by 32 read entries (CT), one copy per lane index: every lane reads its
//   own copy, so lanes at different levels never collide on a bank;
//   then S [L+2][NT] u32, the per-lane stack of Alg. 4's L sets (slot = level+1).
template <int N, bool VS>
struct Layout {
    static constexpr int NT_FIXED = Geo<N, VS>::LAYOUT < 2 ? 1024 : 0;   // lanes per CTA (0 = runtime)
    static constexpr int SST_FIXED = NT_FIXED ? NT_FIXED : ((DLS_UNIFIED && Geo<N, VS>::LAYOUT == 3) ? 1024 : 0);
    // a read entry has 2 (byte layout) or 4 words but always a 16-byte lane stride,
    // so the toggle and read parts of a transition share one address register
    static constexpr int BLK_WORDS = 32 * 8;                  // words per transition block
    // stack entries: the candidate sets of one level, u8 for N <= 8 (layout 0),
    // else u16.  PACK entries share a 32-bit word: entry (slot s, lane t) is byte
    // s * NT * sizeof(SW) + 4 t + sizeof(SW) * (t / (NT / PACK)), so the lanes of a
    // warp always touch 32 different banks (whatever their levels) and slot s of a
    // lane is still element s * NT of an SW array based at the lane's offset
    typedef typename std::conditional<Geo<N, VS>::LAYOUT == 0, uint8_t, uint16_t>::type SW;
    static constexpr int PACK = 4 / (int)sizeof(SW);
    // closure events (CLOSE kernels): a stack of up to cl_cq events per lane,
    // [slot][lane] (cl_cq: as many slots as the launch's shared memory holds,
    // kCqMin .. kCqMax).  The warp looks at the stacks every GROUP steps: once
    // enough lanes hold an event, every lane evaluates (and pops) its newest
    // one; a stack deeper than cl_cq - GROUP forces such rounds until none is,
    // so no stack can overflow during the next group
    static constexpr int GROUP = Geo<N, VS>::LAYOUT == 0 ? 6 : 4;
};

__host__ __device__ inline uint32_t stack_lane_offset(int t, int nt, int sw) {
    return 4u * (uint32_t)t + (uint32_t)sw * (uint32_t)(t / (nt / (4 / sw)));
}

// Rebuild a complete square from the workunit record and the lane's stack and
// append it to p.emit (the optional compact emit of squares for small N).
template <int N, bool VS, class SW>
__device__ __noinline__ void emit_square(const Params &p, int pid, const SW *S, int NT) {
    typedef Geo<N, VS> G;
    DLS_CHECK(pid >= 0 && pid < p.n_prefix, kChkEmit);
    const u64 slot = atomicAdd(p.stats + 7, 1ull);
    if ((long long)slot >= p.emit_cap) return;
    uint8_t *dst = p.emit + slot * (u64)(N * N);
    const uint8_t *rec = p.prefixes + (u64)pid * (u64)(N * N);
    for (int c = 0; c < N * N; ++c) dst[c] = rec[c];
    for (int l = 1; l <= p.L; ++l) {
        const int cell = p.level_cell[l];
        const int pos = __ffs((uint32_t)S[(l + 1) * NT]) - 1;
        // internal bit position -> value (VS: positions >= N/2 hold N-1-(p-N/2))
        const int v = (!VS || pos < G::H) ? pos : N - 1 - (pos - G::H);
        dst[cell] = (uint8_t)v;
        if (VS) dst[(cell / N) * N + (N - 1 - cell % N)] = (uint8_t)(N - 1 - v);
    }
}


// lanes per CTA at most: 1024 for the byte / word-field layouts; 896 for the
// 9- / 10-bit-field layouts, whose larger state needs up to 72 registers
__host__ __device__ constexpr int max_lanes(int layout) { return layout < 2 ? 1024 : 896; }

// CROW (layouts 0 and 1, CLOSE): row r1 has no searched cell, so a closure event is
// the two column words only (8 bytes, twice the event-stack depth) and row r1's
// field is read from a per-lane byte written when the workunit is adopted
template <int N, bool VS, bool EMIT, bool CLOSE, bool LOOK = false, bool CROW = false>
__global__ void __launch_bounds__(max_lanes(Geo<N, VS>::LAYOUT), 1)
dls_search_kernel(const __grid_constant__ Params p) {
    typedef Masks<N, VS> M;
    typedef typename M::CT CT;
    typedef Layout<N, VS> LY;
    typedef Close<N, VS> CL;
    // table block of a transition: 32 toggle entries, 32 read entries (16-byte
    // lane stride), then (LOOK) 32 watched-cell entries of 8 bytes
    constexpr int BLKW = LY::BLK_WORDS + (LOOK ? 64 : 0);
    extern __shared__ __align__(16) uint32_t smem[];
    const int L = p.L;
    const int NT = LY::NT_FIXED ? LY::NT_FIXED : (int)blockDim.x;
    // stack slot stride in entries: the lane count, or 1024 for layout 3 (a power
    // of two lets the unified-address step reach a slot with one multiply-add)
    const int SST = LY::SST_FIXED ? LY::SST_FIXED : NT;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    typedef typename LY::SW SW;
    char *const stk = reinterpret_cast<char *>(smem + (L + 2) * BLKW);
    // closure event stacks ([slot][lane], Close::EW words per entry) after the
    // stack (16-byte aligned)
    const uint32_t stack_bytes = (uint32_t)(L + 1 + LY::PACK) * (uint32_t)SST * (uint32_t)sizeof(SW);
    char *const cq_mem = stk + ((stack_bytes + 15u) & ~15u);
    static_assert(!CROW || (CLOSE && Geo<N, VS>::LAYOUT <= 1 && !LOOK && !EMIT), "CROW: byte / word-field layout, closure");
    constexpr uint32_t EW = CROW ? 2u : (uint32_t)CL::EW;                    // words per event
    constexpr int kGroup = CROW ? DLS_GROUP8 : LY::GROUP;                      // steps between looks at the event stacks
    const uint32_t CQSTR = (uint32_t)NT * EW * 4u;                           // bytes per slot
    const uint32_t cq_sa = (uint32_t)__cvta_generic_to_shared(cq_mem);
    const uint32_t cq_lane0 = cq_sa + (uint32_t)tid * EW * 4u;
    uint8_t *const rowf_s = reinterpret_cast<uint8_t *>(cq_mem + (uint32_t)p.cl_cq * CQSTR);   // CROW: row r1's field per lane
    uint32_t cq_w = cq_lane0;          // shared address of this lane's next event slot
    // a lane's stack is deeper than k events iff cq_w > cq_lane0 + k * CQSTR
    const uint32_t cq_high = cq_lane0 + (uint32_t)(p.cl_cq - kGroup) * CQSTR;
    const uint32_t cl_min = (uint32_t)p.cl_min;    // lanes holding an event that start a round
    const uint32_t rsel = (uint32_t)p.cl_rword;

    // byte layout: the 8-byte read entries sit at an 8-byte lane stride (2
    // shared-memory wavefronts per warp instead of the 4 of a 16-byte stride);
    // the other layouts' read entries are 16 bytes
    constexpr bool kRead8 = DLS_READ8 && sizeof(CT) == 8;
    for (int k = tid; k < (L + 2) * 32; k += NT) {
        const Tab &e = p.tab[k >> 5];
        uint32_t *const blk = smem + (k >> 5) * BLKW;
        reinterpret_cast<uint4 *>(blk)[k & 31] = make_uint4(e.w[0], e.w[1], e.w[2], e.w[3]);
        if constexpr (kRead8)
            reinterpret_cast<uint2 *>(blk + 128)[k & 31] = make_uint2(e.w[4], e.w[5]);
        else
            reinterpret_cast<uint4 *>(blk + 128)[k & 31] = make_uint4(e.w[4], e.w[5], e.w[6], e.w[7]);
        if (LOOK) reinterpret_cast<uint2 *>(blk + 256)[k & 31] = make_uint2(p.look_sel[k >> 5][0], p.look_sel[k >> 5][1]);
    }
    // the slots of levels -1 and 0 are read (idle lanes, backtrack from level 1)
    // but never written: they stay 0
    // slot of level l (l = -1 .. L): S[(l + 1) * SST]
    SW *const S = reinterpret_cast<SW *>(stk + stack_lane_offset(tid, SST, (int)sizeof(SW)));
    S[0] = 0u;
    S[SST] = 0u;
    __syncthreads();
    // transition t: Fl[t * kBlk] (toggle part), Cl at +512 bytes (read part)
    constexpr int kBlk = BLKW / 4;                  // block stride in uint4 units

    const uint4 *const Fl = reinterpret_cast<const uint4 *>(smem + BLKW) + lane;
    const CT *const Cl = reinterpret_cast<const CT *>(smem + BLKW + 128 + (kRead8 ? 2 : 4) * lane);
    const char *const Cb = reinterpret_cast<const char *>(Cl);
    const char *const Fb = reinterpret_cast<const char *>(Fl);   // byte view for t-offsets
    // unified-address step (DLS_UNIFIED): shared addresses of the lane's entry of
    // transition 0 and of level L + 1, and the distance from a level's entry to
    // the stack slot S[level * NT]
    constexpr bool kUni = DLS_UNIFIED && (Geo<N, VS>::LAYOUT == 0 || Geo<N, VS>::LAYOUT == 1 || Geo<N, VS>::LAYOUT == 3) &&
                          !LOOK && !EMIT && BLKW * 4 == 1024 && LY::SST_FIXED == 1024;
    constexpr int kSS = sizeof(SW) == 1 ? 0 : 1;     // a stack slot is 1024 << kSS bytes
    static_assert(!CROW || kUni, "CROW kernels use the unified-address step");
    const uint32_t fl_sa = (uint32_t)__cvta_generic_to_shared(Fb);
    const uint32_t x_last = fl_sa + ((uint32_t)L << 10);          // above it: level L + 1
    const uint32_t d_stk = (uint32_t)__cvta_generic_to_shared(S) - (fl_sa << kSS);   // slot = (entry << kSS) + d_stk
    const uint32_t d_rd = (uint32_t)__cvta_generic_to_shared(Cb) - fl_sa;   // entry -> its read part
    // (LOOK) watched-cell entries: 8-byte lane stride after the 1024 bytes of the two parts
    const char *const Lb = reinterpret_cast<const char *>(smem + BLKW + 256) + 8 * lane;

    uint32_t *const pool = p.pool;

    if (lane == 0) {
        atomicAdd(pool + 0, 1u);                   // this warp is active
        __threadfence();
        atomicAdd(pool + 4, 1u);                   // ... and registered
        stamp_first(pool, kStampStart);
    }
    // (lane 0's acc[5] != 0 marks the warp as waiting: it holds the back-off)

    M st;
    st.clear();
    int lvl = 0;           // 0: idle / finished, 1..L: searching level lvl
    uint32_t cur = 0;      // untried candidates at level lvl
    int pid = -1;          // prefix being searched (n_prefix < 2^31)
    uint32_t cnt = 0;      // completions found for pid by this lane since the last flush
    // per-warp accumulators (shared memory, written by lane 0 / shared atomics):
    // [0] squares, [1] nodes, [2] donations, [3] busy lane-bursts,
    // [4] lane-bursts -- keeps them out of the registers of the search loop
    // [5] (lane 0 only): ns between pool polls of this warp while idle (0: not waiting)
    // [6] closure events evaluated
    // [7] the work queue has run dry (warp-uniform flag, kept here rather than in a
    //     register that would be live -- and spilled -- across the DFS loop)
    __shared__ u64 wacc[32][8];
    u64 *const acc = wacc[tid >> 5];
    if (lane < 8) acc[lane] = 0;
    __syncwarp();
    const u64 n_prefix = (u64)p.n_prefix;

    // One round: every lane holding an event evaluates and pops its newest one;
    // the completions go to the lane's own counter.
    auto close_round = [&](uint32_t &cnt_) {
        const bool has = cq_w != cq_lane0;
        if (has) cq_w -= CQSTR;
        uint32_t k;
        if constexpr (CROW) {
            const uint2 w2 = *reinterpret_cast<const uint2 *>(cq_mem + (cq_w - cq_sa));
            k = CL::eval_cols(w2.x, w2.y, (uint32_t)rowf_s[tid], p);
        } else {
            k = CL::eval(reinterpret_cast<const uint32_t *>(cq_mem + (cq_w - cq_sa)), p, rsel);
        }
        cnt_ += has ? k : 0u;
        const unsigned b = __ballot_sync(kFull, has);
        if (lane == 0) acc[6] += (u64)__popc(b);
    };
    auto close_drain = [&](uint32_t &cnt_) {
        while (__any_sync(kFull, cq_w != cq_lane0)) close_round(cnt_);
    };

    for (;;) {
        // ------------------------------------------------ scheduling point
        if (CLOSE) {
            // every pending event belongs to the lane's current workunit: settle
            // them before a lane finishes it (donated subtrees stay within the
            // workunit, so donors and receivers need no drain)
            if (__any_sync(kFull, pid >= 0 && lvl == 0 && cq_w != cq_lane0)) close_drain(cnt);
            if (pid >= 0 && cnt >= 0x80000000u) {
                if (p.counts) atomicAdd(p.counts + (p.parent ? p.parent[pid] : (uint32_t)pid), (u64)cnt);
                atomicAdd(acc + 0, (u64)cnt);
                cnt = 0;
            }
        }
        if (pid >= 0 && lvl == 0) {
            if (p.counts && cnt) atomicAdd(p.counts + (p.parent ? p.parent[pid] : (uint32_t)pid), (u64)cnt);
            if (cnt) atomicAdd(acc + 0, (u64)cnt);
            cnt = 0;
            pid = -1;
        }
        // a lane that receives work sets pid, fills its stack slots 1..split-1 with
        // the assigned values of the path above `split`, and sets `rest` (the
        // untried values of level split); split = 0 marks a fresh workunit
        bool adopt = false;
        int split = 0;
        uint32_t rest = 0;
        bool qempty = *reinterpret_cast<volatile u64 *>(acc + 7) != 0ull;
        if (!qempty) {
            const unsigned idle = __ballot_sync(kFull, pid < 0);
            if (idle) {
                const int leader = __ffs(idle) - 1;
                u64 base = 0;
                if (lane == leader) base = atomicAdd(p.stats + 3, (u64)__popc(idle));
                base = __shfl_sync(kFull, base, leader);
                if (base + (u64)__popc(idle) >= n_prefix) {
                    qempty = true;
                    if (lane == leader) {
                        acc[7] = 1ull;
                        stamp_first(pool, kStampQEmpty);
                    }
                }
                if (pid < 0) {
                    const u64 my = base + (u64)__popc(idle & lt_mask);
                    if (my < n_prefix) { pid = (int)my; adopt = true; }
                }
            }
        }
        if (qempty) {
            const unsigned idle = __ballot_sync(kFull, pid < 0);
            if (idle == kFull) {
                // ---- whole warp idle: take subtrees other warps donated to the
                // device-wide pool, or leave once no warp is active and none is pending
                uint32_t got = 0, h0 = 0, done = 0;
                if (lane == 0) {
                    if (acc[5] == 0) {               // not yet counted as waiting
                        atomicAdd(pool + 1, 1u);
                        __threadfence();
                        atomicSub(pool + 0, 1u);
                        acc[5] = 128;
                    }
                    // poll with loads; atomics only when something is pending
                    if (ld_acquire(pool + 3) != ld_acquire(pool + 2)) {
                        atomicAdd(pool + 0, 1u);           // tentatively active before claiming
                        for (int tries = 0; tries < 8 && !got; ++tries) {
                            const uint32_t h = ld_acquire(pool + 2), t = ld_acquire(pool + 3);
                            const int avail = (int)(t - h);
                            if (avail <= 0) break;
                            const uint32_t k = min(avail, 32);
                            if (atomicCAS(pool + 2, h, h + k) == h) { got = k; h0 = h; }
                        }
                        if (got) atomicSub(pool + 1, 1u);
                        else atomicSub(pool + 0, 1u);
                    }
                    if (!got) {
                        // every warp registered, none active, nothing pending: the
                        // search is complete (only active warps publish subtrees)
                        const uint32_t reg = ld_acquire(pool + 4);
                        __threadfence();
                        const uint32_t a = ld_acquire(pool + 0);
                        __threadfence();
                        done = (reg == p.total_warps && a == 0u && ld_acquire(pool + 2) == ld_acquire(pool + 3)) ? 1u : 0u;
                    }
                }
                got = __shfl_sync(kFull, got, 0);
                h0 = __shfl_sync(kFull, h0, 0);
                done = __shfl_sync(kFull, done, 0);
                if (done) break;
                if (got && lane == 0) acc[5] = 0;    // active again
                if (!got) {
                    if (lane == 0) {
                        const uint32_t ns = (uint32_t)acc[5];
                        __nanosleep(ns);
                        acc[5] = min(ns * 2u, 8192u);
                    }
                    __syncwarp();
                    continue;
                }
                if ((uint32_t)lane < got) {
                    const uint32_t ticket = h0 + lane;
                    const volatile uint32_t *slot = pool + kPoolHeader + (ticket % kPoolSlots) * kSlotWords;
                    while (slot[0] != ticket + 1u) __nanosleep(64);
                    __threadfence();
                    pid = (int)slot[1];
                    const uint32_t w3 = slot[3];
                    split = (int)(w3 & 0xFFFFu);
                    rest = w3 >> 16;
                    DLS_CHECK(pid >= 0 && (u64)pid < n_prefix && split >= 1 && 2 * split <= L && rest != 0u,
                              kChkPoolGet);
                    for (int l = 1; l < split; ++l)
                        S[(l + 1) * SST] = 1u << ((slot[4 + ((l - 1) >> 3)] >> (4 * ((l - 1) & 7))) & 15u);
                    // consumed: the producer of ticket + kPoolSlots may reuse the slot
                    __threadfence();
                    *const_cast<volatile uint32_t *>(slot + 2) = ticket + 1u;
                    adopt = true;
                }
                __syncwarp();
                if (lane == 0) {
                    __threadfence();
                    atomicAdd(pool + 5, got);   // our slots may be reused from now on
                }
            } else {
                // shallowest open level of each busy lane (its untried siblings)
                int dsplit = 0;
                uint32_t drest = 0;
                if (pid >= 0 && lvl > 0) {
                    for (int l = 1; l < lvl && l <= L - p.min_donate; ++l) {
                        const uint32_t s = S[(l + 1) * SST];
                        if (s & (s - 1u)) { dsplit = l; drest = s & (s - 1u); break; }
                    }
                    if (!dsplit && lvl <= L - p.min_donate && (cur & (cur - 1u))) {
                        dsplit = lvl;
                        drest = cur & (cur - 1u);   // keep the lowest for ourselves
                    }
                }
                unsigned donors = __ballot_sync(kFull, dsplit > 0);
                if (idle && donors && p.donate) {
                    // ---- warp-vote donation to the idle lanes of this warp:
                    // k-th idle lane <- k-th donor lane
                    const int pairs = min(__popc(donors), __popc(idle));
                    const int my_rank = __popc(idle & lt_mask);
                    int src = 0;
                    if (pid < 0 && my_rank < pairs) src = __fns(donors, 0, my_rank + 1);
                    const int dn_rank = __popc(donors & lt_mask);
                    const int d_split = __shfl_sync(kFull, dsplit, src);
                    const uint32_t d_rest = __shfl_sync(kFull, drest, src);
                    const int d_pid = __shfl_sync(kFull, pid, src);
                    const bool recv = pid < 0 && my_rank < pairs;
                    const bool give = dsplit > 0 && dn_rank < pairs;
                    DLS_CHECK(!recv || ((donors >> src) & 1u && d_split >= 1 && d_split <= L && d_rest != 0u &&
                                        d_pid >= 0), kChkWarpGive);
                    if (recv) {
                        // copy the donor's path above the split level
                        const SW *const Sd = reinterpret_cast<const SW *>(stk + stack_lane_offset(tid - lane + src, SST, (int)sizeof(SW)));
                        for (int l = 1; l < d_split; ++l) S[(l + 1) * SST] = Sd[(l + 1) * SST];
                    }
                    __syncwarp();
                    if (give) {
                        if (dsplit < lvl) S[(dsplit + 1) * SST] &= 0u - S[(dsplit + 1) * SST];
                        else cur &= 0u - cur;
                        dsplit = 0;
                    }
                    if (lane == 0) acc[2] += (u64)pairs;
                    if (recv) {
                        pid = d_pid;
                        split = d_split;
                        rest = d_rest;
                        adopt = true;
                    }
                    donors = __ballot_sync(kFull, dsplit > 0);
                }
                if (donors && p.donate) {
                    // ---- donors left over: feed the device-wide pool if a warp waits
                    uint32_t feed = 0;
                    if (lane == 0)
                        feed = (ld_acquire(pool + 1) != 0u && (int)(ld_acquire(pool + 3) - ld_acquire(pool + 5)) < (int)kPoolLimit) ? 1u : 0u;
                    feed = __shfl_sync(kFull, feed, 0);
                    if (feed) {
                        // the lane with the shallowest open level donates it
                        // (only subtrees from the upper half of the tree are worth a trip
                        // through global memory)
                        const uint32_t key = (dsplit > 0 && 2 * dsplit <= L) ? ((uint32_t)dsplit << 5) | (uint32_t)lane
                                                                             : 0xFFFFFFFFu;
                        const uint32_t best = __reduce_min_sync(kFull, key);
                        if (best != 0xFFFFFFFFu && (best & 31u) == (uint32_t)lane) {
                            // at most kPoolLimit + (warps in the grid) < kPoolSlots tickets
                            // can be unreleased: each warp publishes at most one per check
                            const uint32_t ticket = atomicAdd(pool + 3, 1u);
                            DLS_CHECK(ticket - ld_acquire(pool + 5) < kPoolSlots && 4 + (dsplit + 6) / 8 <= kSlotWords,
                                      kChkPoolPut);
                            uint32_t *slot = pool + kPoolHeader + (ticket % kPoolSlots) * kSlotWords;
                            // wait until the slot's previous occupant (ticket - kPoolSlots)
                            // has been read completely (its reader stamps w2)
                            const uint32_t prev = ticket >= kPoolSlots ? ticket + 1u - kPoolSlots : 0u;
                            while (ld_acquire(slot + 2) != prev) __nanosleep(32);
                            slot[1] = (uint32_t)pid;
                            slot[3] = (uint32_t)dsplit | (drest << 16);
                            for (int w = 0; w < (dsplit + 6) / 8; ++w) {
                                uint32_t word = 0;
                                for (int k = 0; k < 8; ++k) {
                                    const int l = 1 + w * 8 + k;
                                    if (l < dsplit) word |= (uint32_t)(__ffs(S[(l + 1) * SST]) - 1) << (4 * k);
                                }
                                slot[4 + w] = word;
                            }
                            __threadfence();
                            *(volatile uint32_t *)slot = ticket + 1u;
                            if (dsplit < lvl) S[(dsplit + 1) * SST] &= 0u - S[(dsplit + 1) * SST];
                            else cur &= 0u - cur;
                            atomicAdd(acc + 2, 1ull);
                        }
                    }
                }
            }
        }
        if (adopt) {
            DLS_CHECK(pid >= 0 && (u64)pid < n_prefix && split >= 0 && split <= L, kChkAdopt);
            // rebuild Rows/Columns from the record, then replay the path
            const bool ok = load_prefix<N, VS>(p.prefixes + (u64)pid * (u64)(N * N), p.pat[0], p.pat[1], st);
            if constexpr (CLOSE && Geo<N, VS>::LAYOUT >= 3) {
                if (p.cl_swap_a >= 0) st.swap_rows(p.cl_swap_a, p.cl_swap_b);
            }
            if constexpr (CROW) rowf_s[tid] = (uint8_t)((rsel ? st.R1 : st.R0) >> p.cl_rshift);
            cnt = 0;
            if (split == 0) {                  // a fresh workunit from the queue
                if (!ok) {
                    atomicOr(p.stats + 2, 1ull);
                    lvl = 0;
                    cur = 0;
                } else if (L == 0) {
                    cnt = 1;                   // the record is a complete square
                    lvl = 0;
                    cur = 0;
                } else {
                    lvl = 1;                   // enter level 1: transition 0 reads cell(1)
                    cur = st.cand(Cl[0]);
                }
            } else {                           // a donated subtree
                for (int l = 1; l < split; ++l) {
                    if constexpr (Geo<N, VS>::LAYOUT >= 3)
                        st.toggle(Fl[l * kBlk], Cl[l * kBlk], S[(l + 1) * SST], 0u);
                    else
                        st.toggle(Fl[l * kBlk], S[(l + 1) * SST], 0u);
                }
                lvl = split;
                cur = rest;
            }
        }

        // ------------------------------------------------ kBurst DFS steps
        {
            const unsigned busy = __ballot_sync(kFull, pid >= 0);
            if (lane == 0) { acc[3] += (u64)__popc(busy); acc[4] += 32; }
        }
        uint32_t cnt32 = 0, ent32 = 0;
        if constexpr (kUni) {
        // ---- unified-address step (same step as below, see DLS_UNIFIED)
        asm volatile("" ::: "memory");           // the stack is accessed through asm from here
        uint32_t xq = fl_sa + ((uint32_t)lvl << 10);   // entry of transition lvl == slot of level lvl-1 (+ d_stk)
        // address of the stack slot of level lvl-1 (= slot `lvl`), carried from step to step
        uint32_t sa = (xq << kSS) + d_stk;
        // x + k on the FMA pipe (one * k + x) or as a plain add
        const uint32_t one = DLS_FMA_ADDS ? p.one : 1u;
        auto addk = [&](uint32_t x, uint32_t k) { return one * k + x; };
        for (int s0 = 0; s0 < kBurst; s0 += (CLOSE ? kGroup : 8)) {
#pragma unroll
        for (int s = 0; s < (CLOSE ? kGroup : 8); ++s) {
            const bool dn = cur != 0u;
            uint32_t sp;                                   // L of level lvl-1
            if constexpr (kSS == 0)
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(sp) : "r"(sa));
            else
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(sp) : "r"(sa));
            const uint32_t bb = sp & (0u - sp);            // its lowest bit: the value assigned there
            const uint32_t sibs = sp - bb;                 // L &= L-1
#if DLS_STEP_V2
            // the level this step (re)assigns holds X: level lvl's candidates on a
            // descend, the untried siblings of level lvl-1 otherwise; empty =
            // plain backtrack.  One select, one lowest-bit isolation.
            const uint32_t X = dn ? cur : sibs;
            const bool adv = X != 0u;
            const uint32_t x = X & (0u - X);
            DLS_CHECK(xq >= fl_sa && xq <= fl_sa + ((uint32_t)(L + 1) << 10) && (!dn || xq <= fl_sa + ((uint32_t)L << 10)) &&
                      (xq > fl_sa || !adv), kChkStep);
            uint32_t xt = xq;                              // transition t = dn ? lvl : lvl - 1
            if (!dn) xt = addk(xq, 0u - 1024u);
#else
            const uint32_t b = cur & (0u - cur);          // isolate rightmost 1-bit
            const uint32_t sb = sibs & (0u - sibs);
            const bool mv = !dn && sibs != 0u;
            const bool adv = dn || mv;
            const uint32_t X = dn ? cur : sibs;
            DLS_CHECK(xq >= fl_sa && xq <= fl_sa + ((uint32_t)(L + 1) << 10) && (!dn || xq <= fl_sa + ((uint32_t)L << 10)) &&
                      (xq > fl_sa || (!dn && !mv)), kChkStep);
            const uint32_t xt = dn ? xq : addk(xq, 0u - 1024u);   // transition t = dn ? lvl : lvl - 1
#endif
            uint4 f;
            CT cs;
            asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(f.x), "=r"(f.y), "=r"(f.z), "=r"(f.w) : "r"(xt));
            if constexpr (sizeof(CT) == 16)
                asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+512];" : "=r"(cs.x), "=r"(cs.y), "=r"(cs.z), "=r"(cs.w) : "r"(xt));
            else if constexpr (kRead8)
                asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cs.x), "=r"(cs.y) : "r"(one * d_rd + xt));
            else
                asm("ld.shared.v2.u32 {%0, %1}, [%2+512];" : "=r"(cs.x), "=r"(cs.y) : "r"(xt));
#if DLS_STEP_V2
            if constexpr (Geo<N, VS>::LAYOUT == 3) {
                uint32_t d = x;
                if (!dn) d = x - bb;
                st.toggle_d(f, cs, d);                     // mark / unmark
            } else if constexpr (VS) {
                st.toggle(f, x, dn ? 0u : bb);
            } else {
                uint32_t d = x;
                if (!dn) d = x - bb;
                st.toggle_d(f, d, d);
            }
            const uint32_t c = st.cand(cs);
            uint32_t xn = xt;                              // level nl = max(t + adv, 0)
            if (adv) xn = addk(xt, 1024u);
            xn = max(xn, fl_sa);
#else
            if constexpr (Geo<N, VS>::LAYOUT == 3) {
                st.toggle_d(f, cs, dn ? b : sb - bb);
            } else if constexpr (VS) {
                st.toggle(f, dn ? b : sb, dn ? 0u : bb);
            } else {
                const uint32_t d = dn ? b : sb - bb;
                st.toggle_d(f, d, d);
            }
            const uint32_t c = st.cand(cs);
            const uint32_t xn = max(adv ? addk(xt, 1024u) : xt, fl_sa);   // level nl = max(t + adv, 0)
#endif
            sa = (xn << kSS) + d_stk;                      // the slot the step writes and the next one reads
            if constexpr (kSS == 0) {
                if (adv) asm volatile("st.shared.u8 [%0], %1;" :: "r"(sa), "r"(X));
            } else {
                if (adv) asm volatile("st.shared.u16 [%0], %1;" :: "r"(sa), "r"(X));
            }
            if (!CLOSE) cnt32 += xn > x_last ? 1u : 0u;
            ent32 += adv ? 1u : 0u;
            cur = adv ? c : 0u;
            xq = xn;
            if constexpr (CROW) {
                asm volatile("{\n\t.reg .pred ev;\n\tsetp.gt.u32 ev, %1, %2;\n\t"
                             "@ev st.shared.v2.u32 [%0], {%4, %5};\n\t"
                             "@ev mad.lo.u32 %0, %6, %3, %0;\n\t}"
                             : "+r"(cq_w) : "r"(xn), "r"(x_last), "r"(CQSTR), "r"(st.C0), "r"(st.C1), "r"(one));
            } else if constexpr (CLOSE) {
                const uint4 w = CL::pack(st, rsel);
                asm volatile("{\n\t.reg .pred ev;\n\tsetp.gt.u32 ev, %1, %2;\n\t"
                             "@ev st.shared.v4.u32 [%0], {%4, %5, %6, %7};\n\t"
                             "@ev mad.lo.u32 %0, %8, %3, %0;\n\t}"
                             : "+r"(cq_w) : "r"(xn), "r"(x_last), "r"(CQSTR), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w), "r"(one));
            }
        }
            if constexpr (CROW && DLS_ROUNDS_ON_FULL) {
                // deep stacks (8-byte events): the look is one vote -- rounds start
                // when some stack nears its depth and go on while enough lanes hold
                // an event (by then most do)
                if (__any_sync(kFull, cq_w > cq_high)) {
                    unsigned red;
                    do {
                        close_round(cnt32);
                        red = __reduce_add_sync(kFull, (cq_w != cq_lane0 ? 1u : 0u) + (cq_w > cq_high ? 1024u : 0u));
                    } while (red >= cl_min);
                }
            } else if constexpr (CLOSE) {
                const unsigned pk = (cq_w != cq_lane0 ? 1u : 0u) + (cq_w > cq_high ? 1024u : 0u);
                unsigned red = __reduce_add_sync(kFull, pk);
                if (red >= cl_min) {
                    close_round(cnt32);
                    while (__any_sync(kFull, cq_w > cq_high)) close_round(cnt32);
                }
            }
        }
        lvl = (int)((xq - fl_sa) >> 10);
        asm volatile("" ::: "memory");
        } else {
        for (int s0 = 0; s0 < kBurst; s0 += (CLOSE ? kGroup : 8)) {
#pragma unroll
        for (int s = 0; s < (CLOSE ? kGroup : 8); ++s) {
            const bool dn = cur != 0u;                     // descend: cell(lvl) has candidates
            const uint32_t b = cur & (0u - cur);          // isolate rightmost 1-bit
            const int t = dn ? lvl : lvl - 1;              // toggle at cell(t), then read cell(t+1)
            SW *const sl = S + lvl * SST;                   // slot of level lvl-1
            const uint32_t sp = *sl;                       // its L (lowest bit = assigned value)
            const uint32_t bb = sp & (0u - sp);
            const uint32_t sibs = sp - bb;                 // L &= L-1
            const uint32_t sb = sibs & (0u - sibs);        // next value of level lvl-1
            const bool mv = !dn && sibs != 0u;             // advance: re-assign level lvl-1
            DLS_CHECK(lvl >= 0 && lvl <= L + 1 && (!dn || lvl <= L) && (lvl > 0 || (!dn && !mv)), kChkStep);
            if constexpr (!DLS_ONE_STORE) {
                if (dn) sl[SST] = cur;                      // push L of level lvl
                if (mv) sl[0] = sibs;
            }
            const int toff = t * (BLKW * 4);     // byte offset of transition t
            const char *const tp = Fb + toff;              // one address for both parts
            const uint4 f = *reinterpret_cast<const uint4 *>(tp);
            const CT cs = *reinterpret_cast<const CT *>(kRead8 ? Cb + toff : tp + 512);
            if constexpr (Geo<N, VS>::LAYOUT >= 3) {
                st.toggle_d(f, cs, dn ? b : sb - bb);                             // mark / unmark
            } else if constexpr (VS || Geo<N, VS>::LAYOUT == 2) {
                st.toggle(f, dn ? b : sb, dn ? 0u : bb);                          // mark / unmark
            } else {
                const uint32_t d = dn ? b : sb - bb;                              // mark / unmark
                st.toggle_d(f, d, d);
            }
            uint32_t c = st.cand(cs);                     // AllN ^ (Rows | Columns) of cell(t+1)
            if constexpr (LOOK) {
                // lookahead: a watched cell left without candidates cuts the branch
                const uint2 lk = *reinterpret_cast<const uint2 *>(Lb + toff);
                const uint32_t cw = st.cand(make_uint4(0u, 0u, lk.x, lk.y));
                c = cw ? c : 0u;
            }
            const bool adv = dn || mv;
            const int nl = max(t + (adv ? 1 : 0), 0);
            // level L+1 is virtual: reaching it completes a square (P:93
            // SquaresCnt++); its "cell" reads full row/column fields, so c = 0 there
            if constexpr (DLS_ONE_STORE) {
                // the slot a push (slot lvl+1) or an advance (slot lvl) writes is
                // slot nl in both cases: the address the next step loads from
                if (adv) S[nl * SST] = (SW)(dn ? cur : sibs);
            }
            if (!CLOSE) cnt32 += nl > L ? 1u : 0u;    // (CLOSE: the closure rounds add to cnt32)
            if (EMIT && nl > L) emit_square<N, VS, SW>(p, pid, S, SST);
            ent32 += adv ? 1u : 0u;
            cur = adv ? c : 0u;
            lvl = nl;
            if constexpr (CLOSE) {
                // level L+1 is a closure event: append the state to the lane's
                // queue -- two predicated instructions, no branch, no vote
                const uint4 w = CL::pack(st, rsel);
                if constexpr (Geo<N, VS>::LAYOUT != 4) {
                    asm volatile("{\n\t.reg .pred ev;\n\tsetp.gt.s32 ev, %1, %2;\n\t"
                                 "@ev st.shared.v4.u32 [%0], {%4, %5, %6, %7};\n\t"
                                 "@ev add.u32 %0, %0, %3;\n\t}"
                                 : "+r"(cq_w) : "r"(nl), "r"(L), "r"(CQSTR), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w));
                } else {
                    asm volatile("{\n\t.reg .pred ev;\n\tsetp.gt.s32 ev, %1, %2;\n\t"
                                 "@ev st.shared.v4.u32 [%0], {%4, %5, %6, %7};\n\t"
                                 "@ev st.shared.u32 [%0+16], %8;\n\t"
                                 "@ev add.u32 %0, %0, %3;\n\t}"
                                 : "+r"(cq_w) : "r"(nl), "r"(L), "r"(CQSTR), "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w),
                                   "r"(CL::pack_row(st, rsel)));
                }
            }
        }
            if constexpr (CLOSE) {
                // one reduction carries both tests: lanes holding an event (< 1024)
                // and 1024 per stack that could overflow during the next group
                const unsigned pk = (cq_w != cq_lane0 ? 1u : 0u) + (cq_w > cq_high ? 1024u : 0u);
                unsigned red = __reduce_add_sync(kFull, pk);
                if (red >= cl_min) {
                    close_round(cnt32);
                    while (__any_sync(kFull, cq_w > cq_high)) close_round(cnt32);
                }
            }
        }
        }   // generic step
        cnt += cnt32;
        if (cnt >= 0x80000000u) {          // flush before 32 bits could overflow
            if (p.counts) atomicAdd(p.counts + (p.parent ? p.parent[pid] : (uint32_t)pid), (u64)cnt);
            atomicAdd(acc + 0, (u64)cnt);
            cnt = 0;
        }
        const uint32_t wn = __reduce_add_sync(kFull, ent32);
        if (lane == 0) acc[1] += (u64)wn;
    }

    DLS_CHECK(lvl == 0 && pid < 0 && cnt == 0u && cur == 0u && S[0] == 0u && S[SST] == 0u, kChkExit);
    // ------------------------------------------------ block reduction, 1 atomic per block
    __syncthreads();
    if (tid == 0) {
        u64 a[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int w = 0; w < NT / 32; ++w)
            for (int k = 0; k < 7; ++k) a[k] += wacc[w][k];
        atomicAdd(p.stats + 0, a[0]);   // squares
        atomicAdd(p.stats + 1, a[1]);   // nodes (assignments, leaves included)
        atomicAdd(p.stats + 4, a[2]);   // donations
        atomicAdd(p.stats + 5, a[3]);   // busy lane-bursts
        atomicAdd(p.stats + 6, a[4]);   // lane-bursts
        atomicAdd(p.stats + 8, a[6]);   // closure events
        if (!EMIT) atomicMax(p.stats + 7, (u64)ld_acquire(pool + 3));   // subtrees published to the pool
        stamp_first(pool, kStampFirstExit);
        atomicMax(reinterpret_cast<u64 *>(pool + kStampLastExit), globaltimer());
    }
}

typedef void (*KernelFn)(Params);

// close: 0 = plain search, 1 = closure, 2 = closure with column-only events (CROW)
template <int N, bool VS>
KernelFn kernel_for(bool emit, int close, bool look = false) {
    if constexpr (N == 9 && !VS) {
        if (look && !emit) return close ? dls_search_kernel<N, VS, false, true, true> : dls_search_kernel<N, VS, false, false, true>;
    }
    if constexpr (DLS_UNIFIED && Geo<N, VS>::LAYOUT <= 1) {
        if (!emit && close == 2) return dls_search_kernel<N, VS, false, true, false, true>;
    }
    return emit ? dls_search_kernel<N, VS, true, false>
                : (close ? dls_search_kernel<N, VS, false, true> : dls_search_kernel<N, VS, false, false>);
}

KernelFn pick_kernel(int n, bool vs, bool emit, int close, bool look) {
    switch (n) {
        case 1: return kernel_for<1, false>(emit, close);
        case 2: return vs ? kernel_for<2, true>(emit, close) : kernel_for<2, false>(emit, close);
        case 3: return kernel_for<3, false>(emit, close);
        case 4: return vs ? kernel_for<4, true>(emit, close) : kernel_for<4, false>(emit, close);
        case 5: return kernel_for<5, false>(emit, close);
        case 6: return vs ? kernel_for<6, true>(emit, close) : kernel_for<6, false>(emit, close);
        case 7: return kernel_for<7, false>(emit, close);
        case 8: return vs ? kernel_for<8, true>(emit, close) : kernel_for<8, false>(emit, close);
        case 9: return kernel_for<9, false>(emit, close, look);
        case 10: return vs ? kernel_for<10, true>(emit, close) : kernel_for<10, false>(emit, close);
        default: return nullptr;
    }
}

int cuda_fail(cudaError_t e, const char *what) {
    dls::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DLS_E_CUDA;
}

// Host mirror of the device layouts: the per-transition table entries.
int layout_of(int n, bool vs) {
    const int h = n / 2;
    const int rf = vs ? (h > 0 ? h : 1) : n, cf = n, nc = vs ? h : n;
    const int rpw32 = 32 / rf, cpw32 = 32 / cf;
    const bool fits2 = (n + rpw32 - 1) / rpw32 <= 2 && (nc + cpw32 - 1) / cpw32 <= 2;
    return n <= 8 ? 0
         : fits2 ? 1
         : (n == 9 && !vs && DLS_LAYOUT9 == 3) ? 3
         : (n == 10 && !vs && DLS_LAYOUT10 == 4) ? 4 : 2;
}

// swap_a / swap_b (layouts 3, 4; -1: none): these two rows trade their fields
// (Params::cl_swap_a).
void fill_tab(int n, bool vs, const std::vector<int> &level_cells, Tab *tab, int swap_a = -1, int swap_b = -1) {
    const int L = (int)level_cells.size();
    const int lay = layout_of(n, vs);
    const bool bytes = lay == 0;
    const int h = n / 2;
    const int rf = vs ? (h > 0 ? h : 1) : n, cf = n;
    const int rpw = 64 / rf, cpw = 64 / cf;
    const int rpw32 = 32 / rf, cpw32 = 32 / cf;
    auto cell_of = [&](int l) { return level_cells[l - 1]; };   // level l = 1..L
    auto slot = [&](int i) { return (lay == 3 || lay == 4) ? (i == swap_a ? swap_b : (i == swap_b ? swap_a : i)) : i; };
    for (int t = -1; t <= L; ++t) {
        Tab &e = tab[t + 1];
        std::memset(&e, 0, sizeof(e));
        if (t >= 1) {                       // toggle part: cell(t)
            const int i = slot(cell_of(t) / n), j = cell_of(t) % n;
            if (bytes) {
                (i < 4 ? e.w[0] : e.w[1]) = 1u << (8 * (i & 3));
                (j < 4 ? e.w[2] : e.w[3]) = 1u << (8 * (j & 3));
            } else if (lay == 1) {
                (i / rpw32 == 0 ? e.w[0] : e.w[1]) = 1u << ((i % rpw32) * rf);
                (j / cpw32 == 0 ? e.w[2] : e.w[3]) = 1u << ((j % cpw32) * cf);
            } else if (lay == 3) {
                e.w[i / 3] = 1u << ((i % 3) * n);
                e.w[3 + j / 3] = 1u << ((j % 3) * n);
            } else if (lay == 4) {
                if (i == 0) e.w[6] += 1u << n;
                else e.w[(i - 1) / 3] = 1u << (((i - 1) % 3) * n);
                if (j == n - 1) e.w[6] += 1u;
                else e.w[3 + j / 3] = 1u << ((j % 3) * n);
            } else {
                e.w[0] = (uint32_t)((i % rpw) * rf);
                e.w[1] = (uint32_t)(i / rpw);
                e.w[2] = (uint32_t)((j % cpw) * cf);
                e.w[3] = (uint32_t)(j / cpw);
            }
        }
        if (t + 1 >= 1 && L >= 1) {         // read part: cell(t+1); for t = L the virtual
            // level L+1 reads row 0 (assigned in every record, hence full), so its
            // candidate set is empty
            const int cl = std::min(t + 1, L);
            const int i = t + 1 > L ? 0 : slot(cell_of(cl) / n), j = cell_of(cl) % n;
            if (bytes) {
                e.w[4] = (uint32_t)i;
                e.w[5] = (uint32_t)j;
            } else if (lay == 1) {
                e.w[4] = (uint32_t)(32 * (i / rpw32) + (i % rpw32) * rf);
                e.w[5] = (uint32_t)(32 * (j / cpw32) + (j % cpw32) * cf);
            } else if (lay == 3) {
                e.w[6] = (uint32_t)((i % 3) * n) | (uint32_t)(i / 3) << 5;
                e.w[7] = (uint32_t)((j % 3) * n) | (uint32_t)(j / 3) << 5;
            } else if (lay == 4) {
                const uint32_t rs = i == 0 ? (uint32_t)n | 3u << 5 : (uint32_t)(((i - 1) % 3) * n) | (uint32_t)((i - 1) / 3) << 5;
                const uint32_t cs = j == n - 1 ? 3u << 5 : (uint32_t)((j % 3) * n) | (uint32_t)(j / 3) << 5;
                e.w[7] = rs | cs << 16;
            } else {
                e.w[4] = (uint32_t)((i % rpw) * rf);
                e.w[5] = (uint32_t)(i / rpw);
                e.w[6] = (uint32_t)((j % cpw) * cf);
                e.w[7] = (uint32_t)(j / cpw);
            }
        }
    }
}

// Everything a launch needs that depends only on (plan, depth).
// Two-row closure level of a plan below depth-`depth` records (DESIGN.md "Tail
// closure"): the first search level l >= 1 after which exactly two rows r1 < r2
// have empty cells, in the same columns and off both diagonals, and the plan
// covers every empty cell.  Fills the closure fields of prm and returns l, or
// returns -1 (no closure: a truncated plan, e.g. dls_count_cells; the condition
// already holds at the records; the 64-bit A/B layout; DLS_CLOSE=0).
int closure_level(const dls::Plan &plan, int depth, Params *prm) {
    const int n = plan.n;
    const bool vs = plan.vs;
    const int steps = (int)plan.cells.size();
    const int lay = layout_of(n, vs);
    if (lay == 2 || n < 3) return -1;
    if (const char *e = getenv("DLS_CLOSE"))
        if (atoi(e) == 0) return -1;
    std::vector<uint8_t> empty(n * n, 1);
    auto take = [&](int c) {
        empty[c] = 0;
        if (vs) empty[(c / n) * n + (n - 1 - c % n)] = 0;
    };
    for (int c = 0; c < n * n; ++c)
        if (plan.pre[c]) empty[c] = 0;
    for (int s = 0; s < depth; ++s) take(plan.cells[s]);
    {   // the plan must cover every cell: completions, not partial assignments
        std::vector<uint8_t> e2 = empty;
        for (int s = depth; s < steps; ++s) {
            const int c = plan.cells[s];
            e2[c] = 0;
            if (vs) e2[(c / n) * n + (n - 1 - c % n)] = 0;
        }
        for (int c = 0; c < n * n; ++c)
            if (e2[c]) return -1;
    }
    for (int l = 0; l <= steps - depth; ++l) {
        if (l > 0) take(plan.cells[depth + l - 1]);
        int rows[3], nr = 0;
        for (int i = 0; i < n && nr < 3; ++i)
            for (int j = 0; j < n; ++j)
                if (empty[i * n + j]) { rows[nr++] = i; break; }
        if (nr != 2) continue;
        const int r1 = rows[0], r2 = rows[1];
        bool ok = true;
        uint32_t open = 0;
        for (int j = 0; j < n && ok; ++j) {
            const bool e1 = empty[r1 * n + j], ee2 = empty[r2 * n + j];
            if (e1 != ee2) ok = false;
            if (e1 && (r1 == j || r1 + j == n - 1 || r2 == j || r2 + j == n - 1)) ok = false;
            if (e1 && (!vs || 2 * j < n - 1)) open |= 1u << j;
        }
        if (!ok) continue;
        if (l == 0) return -1;       // already closable at the records: plain search
        const int h = n / 2, rf = vs ? (h > 0 ? h : 1) : n, rpw32 = 32 / rf, cpw32 = 32 / n;
        // row r1's word in the mask layout (the closure reads row r1 from it)
        // (layouts 3, 4: row r1 trades places with a row of word R[2], so the step's
        // event store always takes R[2]; a row slot below is the row's place after that)
        int rword = 0, swap_a = -1, swap_b = -1;
        if (lay == 3 || lay == 4) {
            if (r1 == 0) return -1;                          // (row 0 is assigned in every record)
            const int first = lay == 3 ? 6 : 7;              // rows of word R[2]: first .. first + 2
            if (r1 < first) {
                swap_a = r1;
                swap_b = first == r2 ? first + 1 : first;
            }
        }
        auto slot = [&](int i) { return i == swap_a ? swap_b : (i == swap_b ? swap_a : i); };
        const int s1 = slot(r1);                              // row r1's place
        switch (lay) {
            case 0: rword = r1 >= 4; break;
            case 1: rword = r1 / rpw32; break;
            default: rword = 2;
        }
        // walk back over forced cells just before level l (up to 2): the closure
        // assigns them itself.  A cell qualifies if its row or column has every
        // other cell assigned before it (one candidate), it lies in neither r1 nor
        // r2, and (layouts 3, 4) its row shares row r1's word.
        int nf = 0, fcell[2];
        {
            auto assigned_before = [&](int q, int cell) {
                // assigned a priori, in the records, or at a level < q
                if (plan.pre[cell]) return true;
                for (int s2 = 0; s2 < depth + q - 1; ++s2) {
                    const int c2 = plan.cells[s2];
                    if (c2 == cell || (vs && (c2 / n) * n + (n - 1 - c2 % n) == cell)) return true;
                }
                return false;
            };
            // opt-in (DLS_CLOSE_FORCED=1): on DLS8 it trades 2 steps per level-30
            // node for twice the closure events, and loses (590 -> 703 ms)
            const char *ef = getenv("DLS_CLOSE_FORCED");
            const bool walk = ef && atoi(ef) != 0;
            while (walk && nf < 2 && l - 1 >= 1) {
                const int cell = plan.cells[depth + l - 1];
                const int i = cell / n, j = cell % n;
                if (i == r1 || i == r2) break;
                if ((lay == 3 || lay == 4) && (lay == 3 ? slot(i) / 3 : (i == 0 ? 3 : (slot(i) - 1) / 3)) != rword) break;
                int rowc = 0, colc = 0;
                for (int k = 0; k < n; ++k) {
                    if (k != j && assigned_before(l, i * n + k)) ++rowc;
                    if (k != i && assigned_before(l, k * n + j)) ++colc;
                }
                if (vs || (rowc != n - 1 && colc != n - 1)) break;   // (VS: not needed by our plans)
                fcell[nf++] = cell;
                --l;
            }
        }
        const int nc = vs ? h : n;                                   // tracked columns
        const int em = vs ? std::max(h - 1, 1) : std::max(n - 2, 1);  // CloseBase::EM
        const int E = __builtin_popcount(open);
        if (E > em || E == nc) return -1;
        int pad = 0;                                                 // a complete column
        while (open >> pad & 1u) ++pad;
        auto sel = [&](int j) -> uint32_t {
            switch (lay) {
                case 0: return (uint32_t)j;
                case 1: return (uint32_t)(32 * (j / cpw32) + (j % cpw32) * n);
                case 3: return (uint32_t)((j % 3) * n) | (uint32_t)(j / 3) << 5;
                default: return j == n - 1 ? 3u << 5 : (uint32_t)((j % 3) * n) | (uint32_t)(j / 3) << 5;
            }
        };
        int k = 0;
        for (int j = 0; j < nc; ++j)
            if (open >> j & 1u) prm->cl_sel[k++] = sel(j);
        while (k < 10) prm->cl_sel[k++] = sel(pad);
        prm->close = 1;
        {   // column-only events (CROW kernels): byte layout, unified step, no
            // forced-cell walk, and no searched cell in row r1
            bool row_const = lay <= 1 && DLS_UNIFIED && nf == 0;
            for (int s2 = depth; s2 < depth + l && row_const; ++s2)
                if (plan.cells[s2] / n == r1) row_const = false;
            if (const char *e8 = getenv("DLS_CLOSE_ROW8"))
                if (atoi(e8) == 0) row_const = false;             // A/B: 16-byte events
            if (row_const) prm->close = 2;
        }
        prm->cl_swap_a = swap_a;
        prm->cl_swap_b = swap_b;
        prm->cl_min = kCloseMinLanes;
        if (const char *e = getenv("DLS_CLOSE_MIN")) prm->cl_min = std::min(32, std::max(1, atoi(e)));   // tuning
        prm->cl_open = open;
        prm->cl_E = E;
        prm->cl_nf = nf;
        for (int k = 0; k < nf; ++k) {      // apply in plan order: the earlier cell first
            Tab t3[3];
            fill_tab(n, vs, std::vector<int>{fcell[nf - 1 - k]}, t3, swap_a, swap_b);
            prm->cl_fread[k] = t3[1];       // transition 0 reads cell(1)
            prm->cl_ftog[k] = t3[2];        // transition 1 toggles cell(1)
        }
        switch (lay) {
            case 0: prm->cl_rword = r1 >= 4; prm->cl_rshift = 8 * (r1 & 3); break;
            case 1: prm->cl_rword = r1 / rpw32; prm->cl_rshift = (r1 % rpw32) * rf; break;
            case 3: prm->cl_rword = 2; prm->cl_rshift = n * (s1 % 3); break;
            default: prm->cl_rword = 2; prm->cl_rshift = n * ((s1 - 1) % 3);
        }
        return l;
    }
    return -1;
}

int prepare_plan(const dls::Plan &plan, int depth, Params *prm, bool allow_close = true) {
    const int n = plan.n;
    const bool symmetric = plan.vs;
    const int steps = (int)plan.cells.size();
    {   // the virtual last level reads row 0: it must be assigned in every record
        const auto first = plan.cells.begin(), last = plan.cells.begin() + std::min(depth, steps);
        for (int j = 0; j < n; ++j) {
            const int jm = symmetric ? n - 1 - j : j;   // VS plans list left-half cells only
            if (!plan.pre[j] && std::find(first, last, j) == last && std::find(first, last, jm) == last) {
                dls::set_error("dls_count: row 0 must be assigned in the records");
                return DLS_E_ARG;
            }
        }
    }
    if (depth < plan.diag_depth || depth > steps) {
        dls::set_error("dls_count: depth must satisfy diag_depth <= depth <= n_steps");
        return DLS_E_ARG;
    }
    std::memset(prm, 0, sizeof(*prm));
    prm->cl_swap_a = prm->cl_swap_b = -1;
    prm->L = steps - depth;
    if (allow_close) {
        const int lc = closure_level(plan, depth, prm);
        if (lc >= 0) prm->L = lc;
    }
    std::vector<int> level_cells(plan.cells.begin() + depth, plan.cells.begin() + depth + prm->L);
    fill_tab(n, symmetric, level_cells, prm->tab, prm->cl_swap_a, prm->cl_swap_b);
    // lookahead, DLS N = 9 only, opt-in: DLS_LOOKAHEAD=a-b applies it
    // after the plan steps a..b (1-based, Fig. 1 numbering; the paper: 51-60).
    // The watched cell of a step assigning (i, j) is the first later plan cell
    // (after the next one) in row i or column j.
    if (const char *la = getenv("DLS_LOOKAHEAD")) {
        int a = 0, b = -1;
        if (n == 9 && !symmetric && layout_of(n, symmetric) == 3 && sscanf(la, "%d-%d", &a, &b) == 2 && a <= b) {
            prm->look = 1;
            for (int t = -1; t <= prm->L; ++t) {
                prm->look_sel[t + 1][0] = prm->tab[t + 1].w[6];   // default: cell(t+1) itself
                prm->look_sel[t + 1][1] = prm->tab[t + 1].w[7];
                const int step = depth + t;                        // plan step of cell(t), 1-based
                if (t < 1 || t >= prm->L || step < a || step > b) continue;
                const int c0 = plan.cells[depth + t - 1], i0 = c0 / n, j0 = c0 % n;
                for (size_t q = depth + t + 1; q < plan.cells.size(); ++q) {
                    const int c = plan.cells[q];
                    if (c / n != i0 && c % n != j0) continue;
                    Tab t3[3];
                    fill_tab(n, symmetric, std::vector<int>{c}, t3, prm->cl_swap_a, prm->cl_swap_b);
                    prm->look_sel[t + 1][0] = t3[1].w[6];
                    prm->look_sel[t + 1][1] = t3[1].w[7];
                    break;
                }
            }
        }
    }
    for (size_t l = 0; l < level_cells.size(); ++l) prm->level_cell[l + 1] = (uint8_t)level_cells[l];
    // assigned-cell pattern of a depth-`depth` prefix
    auto set = [&](int c) { prm->pat[c >> 6] |= 1ull << (c & 63); };
    for (int c = 0; c < n * n; ++c)
        if (plan.pre[c]) set(c);
    for (int s = 0; s < depth; ++s) {
        const int c = plan.cells[s];
        set(c);
        if (symmetric) set((c / n) * n + (n - 1 - c % n));
    }
    prm->donate = 1;
    prm->min_donate = std::max(kMinDonateDepth, prm->L / 3);
    if (const char *e = getenv("DLS_DONATE")) prm->donate = atoi(e);   // 0: no donation (diagnostics)
    if (const char *e = getenv("DLS_MIN_DONATE")) prm->min_donate = std::max(1, atoi(e));   // tuning
    return DLS_OK;
}

int prepare(int n, int symmetric, int fixed_first_row, int depth, Params *prm, bool allow_close = true) {
    dls::Plan plan;
    if (!dls::make_plan(n, symmetric, fixed_first_row, &plan)) {
        dls::set_error("dls_count: unsupported (n, symmetric, fixed_first_row)");
        return DLS_E_ARG;
    }
    return prepare_plan(plan, depth, prm, allow_close);
}

// event slots per lane of the closure kernels: at least kCqMin (= the largest
// GROUP + 2), at most kCqMax
constexpr int kCqMin = 8, kCqMinWide = 6, kCqMax = 20;

// shared memory of a launch; cq = event slots per lane (0: no closure)
size_t smem_bytes(int n, bool vs, int L, int nthreads, int cq, bool look = false, bool crow = false) {
    const int lay = layout_of(n, vs);
    const size_t sw = lay == 0 ? 1 : 2;                       // Layout::SW
    const size_t sst = (lay == 3 && DLS_UNIFIED) ? 1024 : nthreads;   // Layout::SST_FIXED
    const size_t stack = (size_t)(L + 1 + 4 / sw) * sst * sw;
    const size_t base = (size_t)(L + 2) * (look ? 40 : 32) * 32 + ((stack + 15) & ~(size_t)15);
    const size_t ew = crow ? 2 : (lay == 4 ? 8 : 4);          // words per event
    return base + (size_t)cq * nthreads * ew * 4 + (crow ? (size_t)nthreads : 0);   // event stacks (+ row bytes)
}

int launch(int n, bool vs, const Params &prm, cudaStream_t stream) {
    const int close = prm.emit == nullptr ? prm.close : 0;      // 0 / 1 / 2 (column-only events)
    const bool crow = close == 2;
    const bool look = prm.look && prm.emit == nullptr;
    KernelFn fn = pick_kernel(n, vs, prm.emit != nullptr, close, look);
    if (!fn) { dls::set_error("no kernel for this order"); return DLS_E_ARG; }
    cudaError_t e;
    int dev = 0, sms = 0, smem_max = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return cuda_fail(e, "cudaDeviceGetAttribute");
    if ((e = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
        return cuda_fail(e, "cudaDeviceGetAttribute");
    smem_max -= 2048;   // static shared memory of the kernel (per-warp accumulators, 1.75 KB)
    // one persistent CTA per SM with as many lanes as fit (multiple of 32, <= 1024)
    const int lay = layout_of(n, vs);
    int nthreads = max_lanes(lay);         // = the kernel's __launch_bounds__ (layouts 0, 1: fixed)
    // (a multiple of 64, so that the u16 stack's lanes keep distinct banks)
    const int cq_min = !close ? 0 : (crow ? DLS_GROUP8 + 2 : (lay == 0 ? kCqMin : kCqMinWide));
    while (lay >= 2 && nthreads > 64 && smem_bytes(n, vs, prm.L, nthreads, cq_min, look, crow) > (size_t)smem_max) nthreads -= 64;
    int cq = cq_min;
    if (const char *ec = getenv("DLS_CLOSE_CQ")) cq = std::max(cq_min, atoi(ec));   // tuning: cap the depth
    else cq = kCqMax;
    while (cq > cq_min && smem_bytes(n, vs, prm.L, nthreads, cq, look, crow) > (size_t)smem_max) --cq;
    if (!close) cq = 0;
    const size_t smem = smem_bytes(n, vs, prm.L, nthreads, cq, look, crow);
    if (smem > (size_t)smem_max) { dls::set_error("search state does not fit in shared memory"); return DLS_E_ARG; }
    if ((e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return cuda_fail(e, "cudaFuncSetAttribute");
    // one CTA per SM even for few workunits: warps without a workunit start by
    // taking donated subtrees from the device-wide pool
    void *pool = nullptr;
    if ((e = dls::scratch_alloc(&pool, kPoolBytes, stream)) != cudaSuccess) return cuda_fail(e, "scratch_alloc(pool)");
    if ((e = cudaMemsetAsync(pool, 0, kPoolBytes, stream)) != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(pool)");
    Params q = prm;
    q.pool = (uint32_t *)pool;
    q.cl_cq = cq;
    q.one = 1u;
    q.total_warps = (uint32_t)sms * (uint32_t)(nthreads / 32);
    // Cooperative launch: the exit test waits for every warp of the grid to have
    // registered, so all CTAs must be resident at once; the launch guarantees it
    // or fails (e.g. while other work holds SMs) instead of hanging.
    void *args[] = {&q};
    if ((e = cudaLaunchCooperativeKernel((const void *)fn, dim3((unsigned)sms), dim3((unsigned)nthreads), args, smem,
                                         stream)) != cudaSuccess)
        return cuda_fail(e, "kernel launch (cooperative)");
    if (getenv("DLS_TIMING")) {   // end-game timeline of this launch (synchronises)
        u64 st[8];
        cudaMemcpyAsync(st, (uint32_t *)pool + kStampStart, sizeof(st), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        const double t0 = (double)st[0];
        fprintf(stderr, "[launch] n_prefix %lld: queue empty at %.1f ms, first CTA exit %.1f ms, last %.1f ms\n",
                (long long)prm.n_prefix, st[1] ? (st[1] - t0) / 1e6 : -1.0, (st[2] - t0) / 1e6, (st[3] - t0) / 1e6);
    }
    if ((e = cudaFreeAsync(pool, stream)) != cudaSuccess) return cuda_fail(e, "cudaFreeAsync(pool)");
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

#ifdef DLS_CHECKS
extern "C" const char *dls_version(void) { return "dls_b200 0.1.0 sm_100a checked"; }
#else
extern "C" const char *dls_version(void) { return "dls_b200 0.1.0 sm_100a"; }
#endif

extern "C" int dls_count_async(int n, int symmetric, int fixed_first_row, int depth,
                               const uint8_t *d_prefixes, int64_t n_prefix, uint64_t *d_counts,
                               uint64_t *d_stats, void *stream) {
    int rc = have_device();
    if (rc) return rc;
    if (n_prefix < 0 || n_prefix >= (int64_t)1 << 31 || (n_prefix > 0 && !d_prefixes) || !d_stats) {
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

// Device scratch of the synchronous dls_count, cached per device (grow-only) so
// repeated calls do not pay cudaMalloc/cudaFree; the mutex serialises callers.
struct Workspace {
    std::mutex mu;
    void *p = nullptr;
    size_t cap = 0;
};
Workspace g_ws[64];

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// The kernel's error word stats[2]: bit 0 = an inconsistent prefix record, bits
// 8.. = violated internal invariants (checked build only, see DLS_CHECK).
int error_word(u64 w, const char *who) {
    if (w >> 8) {
        char msg[160];
        snprintf(msg, sizeof msg, "%s: internal check failed (mask 0x%llx)", who, (unsigned long long)(w >> 8));
        dls::set_error(msg);
        return DLS_E_CUDA;
    }
    if (w) {
        dls::set_error(std::string(who) + ": some prefix record is not a consistent depth-d prefix");
        return DLS_E_PREFIX;
    }
    return DLS_OK;
}

}  // namespace


namespace dls {

// Scratch device memory (the donation pool, the symmetry-breaking buffers) comes
// from the library's own stream-ordered memory pool, one per device, created on
// first use.  Its release threshold is 1 GB: with the default threshold (0)
// every synchronisation hands the freed memory back to the OS, and that used to
// cost 0.25-1.2 s after the kernel had finished (profiles/r1_e2e_variance.log).
// The process's default pool (PyTorch's cudaMallocAsync backend, other users)
// is left alone.
namespace {
std::once_flag g_pool_once[64];
cudaMemPool_t g_pools[64];
cudaError_t g_pool_status[64];

// this device's pool (created on first use), or the creation error
cudaError_t library_pool(cudaMemPool_t *out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::call_once(g_pool_once[dev & 63], [dev]() {
        cudaMemPoolProps props;
        std::memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaError_t e1 = cudaMemPoolCreate(&g_pools[dev & 63], &props);
        if (e1 == cudaSuccess) {
            uint64_t keep = 1ull << 30;
            if (const char *k = getenv("DLS_POOL_KEEP")) keep = (uint64_t)atoll(k);
            e1 = cudaMemPoolSetAttribute(g_pools[dev & 63], cudaMemPoolAttrReleaseThreshold, &keep);
        }
        g_pool_status[dev & 63] = e1;
    });
    *out = g_pools[dev & 63];
    return g_pool_status[dev & 63];
}
}  // namespace

cudaError_t scratch_alloc(void **ptr, size_t bytes, cudaStream_t stream) {
    cudaMemPool_t mp;
    const cudaError_t e = library_pool(&mp);
    if (e != cudaSuccess) return e;
    return cudaMallocFromPoolAsync(ptr, bytes, mp, stream);
}

// Hand cached scratch above keep_bytes back (after large symmetry-breaking calls).
void scratch_trim(size_t keep_bytes) {
    cudaMemPool_t mp;
    if (library_pool(&mp) == cudaSuccess) cudaMemPoolTrimTo(mp, keep_bytes);
    cudaGetLastError();
}

// dls_count for an arbitrary plan (the standard one, or the hourglass plan of
// the symmetry-broken driver).
int count_records(const Plan &plan, int depth, const uint8_t *prefix_buf, int64_t n_prefix, uint64_t *out_counts,
                  uint64_t *out_total, uint64_t *out_nodes, void *stream, int64_t refine_below) {
    int rc = have_device();
    if (rc) return rc;
    if (n_prefix < 0 || n_prefix >= (int64_t)1 << 31 || (n_prefix > 0 && !prefix_buf)) {
        dls::set_error("dls_count: bad pointers / sizes");
        return DLS_E_ARG;
    }
    const int n = plan.n;
    Params prm;
    if ((rc = prepare_plan(plan, depth, &prm))) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    // DLS_TIMING=1: host-side phase times of this call on stderr
    const bool timing = getenv("DLS_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (!timing) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[count_records] %-22s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
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
    if (refine_below < 0) refine_below = kRefineTarget / 8;
    if (n_prefix > 0 && n_prefix < refine_below && depth + 1 <= steps - kMinSearchLevels && prm.L > 1) {
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
        // stay above the closure level (records at it could not use the closure)
        const int close_pos = depth + prm.L;
        while (cnt < kRefineTarget && d1 + 1 <= steps - kMinSearchLevels && d1 + 1 < close_pos) {
            ++d1;
            cnt = dls::refine(plan, depth, d1, src, n_prefix, nullptr, nullptr, 0, nullptr);
        }
        h_sub.resize((size_t)cnt * nn + 1);
        h_parent.resize((size_t)cnt + 1);
        dls::refine(plan, depth, d1, src, n_prefix, h_sub.data(), h_parent.data(), cnt, &extra_nodes);
        if ((rc = prepare_plan(plan, d1, &prm))) return rc;
        src = h_sub.data();
        n_rec = cnt;
        depth_run = d1;
    }
    const bool refined = depth_run != depth;
    mark("validate + refine");
    if (timing)
        fprintf(stderr, "[count_records] %lld records at depth %d -> %lld at depth %d\n", (long long)n_prefix, depth,
                (long long)n_rec, depth_run);

    const bool counts_host = out_counts && n_prefix > 0 && !is_device_ptr(out_counts);
    const bool stage_records = n_rec > 0 && (refined || !in_dev);
    // workspace layout: stats | counts (host output) | parent map | records
    const size_t off_cnt = align256(DLS_STATS_WORDS * sizeof(u64));
    const size_t off_par = off_cnt + align256(counts_host ? (size_t)n_prefix * sizeof(u64) : 0);
    const size_t off_rec = off_par + align256(refined ? (size_t)n_rec * sizeof(uint32_t) : 0);
    const size_t need = off_rec + (stage_records ? (size_t)n_rec * nn : 0);
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    Workspace &ws = g_ws[dev & 63];
    std::lock_guard<std::mutex> lock(ws.mu);
    if (ws.cap < need) {
        if (ws.p) { cudaStreamSynchronize(s); cudaFree(ws.p); ws.p = nullptr; ws.cap = 0; }
        const size_t cap = need + need / 4;
        if ((e = cudaMalloc(&ws.p, cap)) != cudaSuccess) { ws.p = nullptr; return cuda_fail(e, "cudaMalloc(workspace)"); }
        ws.cap = cap;
    }
    mark("workspace");
    char *const base = (char *)ws.p;
    const uint8_t *d_pre = src;
    if (stage_records) {
        if ((e = cudaMemcpyAsync(base + off_rec, src, (size_t)n_rec * nn, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e, "cudaMemcpyAsync(H2D)");
        d_pre = (const uint8_t *)(base + off_rec);
    }
    u64 *d_counts = counts_host ? (u64 *)(base + off_cnt) : (u64 *)out_counts;
    if (refined &&
        (e = cudaMemcpyAsync(base + off_par, h_parent.data(), (size_t)n_rec * sizeof(uint32_t), cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    u64 *d_stats = (u64 *)base;
    if ((e = cudaMemsetAsync(d_stats, 0, DLS_STATS_WORDS * sizeof(u64), s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync(stats)");
    if (d_counts && n_prefix > 0 &&
        (e = cudaMemsetAsync(d_counts, 0, (size_t)n_prefix * sizeof(u64), s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemsetAsync(counts)");
    if (n_rec > 0) {
        prm.prefixes = d_pre;
        prm.n_prefix = n_rec;
        prm.counts = d_counts;
        prm.parent = refined ? (const uint32_t *)(base + off_par) : nullptr;
        prm.stats = d_stats;
        mark("H2D + memsets enqueued");
        if ((rc = launch(n, plan.vs, prm, s))) { cudaStreamSynchronize(s); return rc; }
        mark("launch enqueued");
    }
    u64 stats[DLS_STATS_WORDS];
    if ((e = cudaMemcpyAsync(stats, d_stats, sizeof(stats), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync(stats)");
    if (counts_host &&
        (e = cudaMemcpyAsync(out_counts, d_counts, (size_t)n_prefix * sizeof(u64), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    mark("search + D2H (sync)");
    if (out_total) *out_total = stats[0];
    if (out_nodes) *out_nodes = stats[1] + (u64)extra_nodes;
    if ((rc = error_word(stats[2] | (bad_prefix ? 1ull : 0ull), "dls_count"))) return rc;
    return DLS_OK;
}

}  // namespace dls

extern "C" int dls_count(int n, int symmetric, int fixed_first_row, int depth,
                         const uint8_t *prefix_buf, int64_t n_prefix, uint64_t *out_counts,
                         uint64_t *out_total, uint64_t *out_nodes, void *stream) {
    dls::Plan plan;
    if (!dls::make_plan(n, symmetric, fixed_first_row, &plan)) {
        dls::set_error("dls_count: unsupported (n, symmetric, fixed_first_row)");
        return DLS_E_ARG;
    }
    return dls::count_records(plan, depth, prefix_buf, n_prefix, out_counts, out_total, out_nodes, stream);
}

extern "C" int dls_search_levels(int n, int symmetric, int fixed_first_row, int depth, int32_t *out_levels) {
    if (!out_levels) { dls::set_error("dls_search_levels: null output"); return DLS_E_ARG; }
    Params prm;
    const int rc = prepare(n, symmetric, fixed_first_row, depth, &prm);
    if (rc) return rc;
    *out_levels = prm.L;
    return DLS_OK;
}

extern "C" int64_t dls_emit(int n, int symmetric, int fixed_first_row, int depth, const uint8_t *d_prefixes,
                            int64_t n_prefix, uint8_t *d_out, int64_t capacity, void *stream) {
    int rc = have_device();
    if (rc) return rc;
    if (n_prefix < 0 || n_prefix >= (int64_t)1 << 31 || (n_prefix > 0 && !d_prefixes) || capacity < 0 ||
        (capacity > 0 && !d_out) || !is_device_ptr(d_prefixes) || (capacity > 0 && !is_device_ptr(d_out))) {
        dls::set_error("dls_emit: bad pointers / sizes (device buffers required)");
        return DLS_E_ARG;
    }
    Params prm;
    if ((rc = prepare(n, symmetric, fixed_first_row, depth, &prm, false))) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    u64 *d_stats = nullptr;
    cudaError_t e = dls::scratch_alloc((void **)&d_stats, DLS_STATS_WORDS * sizeof(u64), s);
    if (e != cudaSuccess) return cuda_fail(e, "scratch_alloc");
    cudaMemsetAsync(d_stats, 0, DLS_STATS_WORDS * sizeof(u64), s);
    prm.prefixes = d_prefixes;
    prm.n_prefix = n_prefix;
    prm.stats = d_stats;
    prm.emit = d_out ? d_out : (uint8_t *)d_stats;   // non-null selects the emit kernel
    prm.emit_cap = capacity;
    if (n_prefix > 0 && (rc = launch(n, symmetric, prm, s))) { cudaFreeAsync(d_stats, s); return rc; }
    u64 stats[DLS_STATS_WORDS];
    cudaMemcpyAsync(stats, d_stats, sizeof(stats), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d_stats, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "dls_emit");
    if ((rc = error_word(stats[2], "dls_emit"))) return (int64_t)rc;
    return (int64_t)stats[0];
}

extern "C" int dls_count_cells(int n, int symmetric, const uint8_t *record, const int32_t *cells, int n_cells,
                               uint64_t *out_total, uint64_t *out_nodes, void *stream) {
    if (n < 1 || n > DLS_MAX_ORDER || (symmetric && n % 2) || !record || n_cells < 0 || (n_cells && !cells)) {
        dls::set_error("dls_count_cells: bad arguments");
        return DLS_E_ARG;
    }
    const int nn = n * n;
    uint8_t pre[DLS_MAX_ORDER * DLS_MAX_ORDER] = {};
    for (int c = 0; c < nn; ++c) pre[c] = record[c] != DLS_EMPTY;
    for (int j = 0; j < n; ++j)
        if (!pre[j]) { dls::set_error("dls_count_cells: row 0 of the record must be assigned"); return DLS_E_ARG; }
    // the listed diagonal cells first (the GPU search tracks rows and columns only)
    std::vector<int> head, rest;
    std::vector<uint8_t> seen(nn, 0);
    for (int k = 0; k < n_cells; ++k) {
        const int c = cells[k];
        if (c < 0 || c >= nn || pre[c] || seen[c] || (symmetric && 2 * (c % n) > n - 1)) {
            dls::set_error("dls_count_cells: cells must be distinct, empty in the record (left half if symmetric)");
            return DLS_E_ARG;
        }
        seen[c] = 1;
        const int i = c / n, j = c % n;
        const bool diag = i == j || i + j == n - 1 || (symmetric && (i == n - 1 - j || i + (n - 1 - j) == n - 1));
        (diag ? head : rest).push_back(c);
    }
    const int dd = (int)head.size();
    head.insert(head.end(), rest.begin(), rest.end());
    dls::Plan plan;
    if (!dls::make_plan_from(n, symmetric, pre, head, &plan)) {
        dls::set_error("dls_count_cells: unsupported order");
        return DLS_E_ARG;
    }
    plan.cells.resize(n_cells);
    plan.forced.resize(n_cells);
    plan.diag_depth = dd;
    // records at the diagonal depth (host), then the GPU search of the other cells
    const int64_t k = dls::refine(plan, 0, dd, record, 1, nullptr, nullptr, 0, nullptr);
    if (k < 0) return (int)k;
    std::vector<uint8_t> recs((size_t)std::max<int64_t>(k, 1) * nn);
    int64_t extra = 0;
    dls::refine(plan, 0, dd, record, 1, recs.data(), nullptr, k, &extra);
    uint64_t total = 0, nodes = 0;
    if (k > 0) {
        if (dd == n_cells) {
            total = (uint64_t)k;
        } else {
            const int rc = dls::count_records(plan, dd, recs.data(), k, nullptr, &total, &nodes, stream);
            if (rc) return rc;
        }
    }
    if (out_total) *out_total = total;
    if (out_nodes) *out_nodes = nodes + (uint64_t)extra;
    return DLS_OK;
}
