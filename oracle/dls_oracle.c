/*
 * dls_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the counting that the
 * B200 path (paper_1709_02599_b200/) performs.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file's
 * shared object.  It shares no code, header, table or helper with the CUDA path.
 *
 * Paper: Kochemazov, Vatutin, Zaikin, "Fast Algorithm for Enumerating Diagonal
 * Latin Squares of Small Order" (arXiv:1709.02599), /root/reference/PAPER.md.
 * Citations "P:<line>" are PAPER.md line numbers.
 *
 * Deliberate choices (north_star): an int array LS[N][N] with -1 for an empty
 * cell; every constraint test is an explicit scan of the row, the column and,
 * when the cell lies on one, the main diagonal / main antidiagonal.  No bit
 * masks anywhere.  Recursion, not an explicit stack.
 *
 * Functions
 *   oracle_plan      -- cell order of P:152-154 (Section 2.3, V-score + forced cells)
 *   oracle_count     -- number of completions of a partial square in a given order
 *                       (Alg. 1/2, with explicit scans instead of the
 *                       occupancy arrays), plus the number of search nodes
 *   oracle_count_levels -- the same, with the nodes split by depth
 *   oracle_prefixes  -- all consistent assignments of the first `depth` cells of an
 *                       order (workunit decomposition)
 *   oracle_squares   -- writes out every completion (for square-by-square checks)
 *   oracle_canonize  -- M-transformations + canonic form of a hourglass design
 *                       (Section 4, Alg. 5)
 *   oracle_classes   -- canonic hourglass designs with class sizes (Alg. 6 outer loops)
 *
 * Vertical symmetry: with vs != 0 only left-half cells (j < N/2 ... or
 * j <= N-1-j) appear in an order; placing v at (i,j) also places N-1-v at
 * (i,N-1-j) and both placements are checked by the same scans.
 *
 * Parity pins: see tests/test_oracle.py (brute force over permutation-row
 * stackings for N<=5, N! x first-row-fixed invariant, VS definition checked square
 * by square, Fig. 1 cell order, hourglass count 22 192 248 of P:436).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXN 16

typedef struct {
    int n;
    int vs;
    int ls[MAXN][MAXN];          /* -1 = empty */
    const int *order;             /* cells as i*n+j */
    int n_order;
    unsigned long long count;
    unsigned long long nodes;
    /* optional outputs */
    int *emit;                    /* prefixes or squares, n*n ints each */
    long long emit_cap;
    long long emitted;
    int emit_depth;               /* stop depth for prefix enumeration (-1 = full) */
    int canon;                    /* 1: at the stop depth canonise (Alg. 5) instead of emitting */
    long long classes;            /* canonical designs found */
    long long *mult_out;          /* their class sizes (up to emit_cap) */
    unsigned long long *level_nodes; /* optional: nodes per depth (assignments of order[k]) */
} oracle_state;

long long oracle_canonize(int n, int vs, const int *g);

/* Does placing value v at (i,j) clash with an already assigned cell of the same
 * row, column, main diagonal (i==j) or main antidiagonal (i+j==n-1)?  (Alg. 2,
 * P:124 "Condition_{i,j}", evaluated by scanning.) */
static int clashes(const oracle_state *s, int i, int j, int v)
{
    int n = s->n, k;
    for (k = 0; k < n; k++) {
        if (k != j && s->ls[i][k] == v) return 1;      /* row i */
        if (k != i && s->ls[k][j] == v) return 1;      /* column j */
    }
    if (i == j) {                                      /* main diagonal */
        for (k = 0; k < n; k++)
            if (k != i && s->ls[k][k] == v) return 1;
    }
    if (i + j == n - 1) {                              /* main antidiagonal */
        for (k = 0; k < n; k++)
            if (k != i && s->ls[k][n - 1 - k] == v) return 1;
    }
    return 0;
}

/* Try to assign v at (i,j) (and, for vs, N-1-v at the mirror cell (i,N-1-j),
 * P:521).  Returns 1 and leaves the assignment in place on success. */
static int place(oracle_state *s, int i, int j, int v)
{
    int n = s->n;
    if (clashes(s, i, j, v)) return 0;
    s->ls[i][j] = v;
    if (s->vs) {
        int jm = n - 1 - j, vm = n - 1 - v;
        if (jm == j) {
            if (vm != v) { s->ls[i][j] = -1; return 0; }
        } else {
            if (s->ls[i][jm] != -1 || clashes(s, i, jm, vm)) { s->ls[i][j] = -1; return 0; }
            s->ls[i][jm] = vm;
        }
    }
    return 1;
}

static void unplace(oracle_state *s, int i, int j)
{
    int n = s->n;
    s->ls[i][j] = -1;
    if (s->vs && n - 1 - j != j) s->ls[i][n - 1 - j] = -1;
}

static void emit_grid(oracle_state *s)
{
    if (s->emit && s->emitted < s->emit_cap) {
        int *dst = s->emit + s->emitted * (long long)s->n * s->n;
        int i, j;
        for (i = 0; i < s->n; i++)
            for (j = 0; j < s->n; j++) dst[i * s->n + j] = s->ls[i][j];
    }
    s->emitted++;
}

/* One nested loop of Alg. 1 per cell of the order: try every value
 * 0..N-1 in increasing order, skip the clashing ones, recurse, undo. */
static void fill(oracle_state *s, int step)
{
    int stop = s->emit_depth >= 0 ? s->emit_depth : s->n_order;
    if (step == stop) {
        s->count++;                      /* SquaresCnt++  */
        if (s->canon) {
            int g[MAXN * MAXN], i, j;
            long long m;
            for (i = 0; i < s->n; i++)
                for (j = 0; j < s->n; j++) g[i * s->n + j] = s->ls[i][j];
            m = oracle_canonize(s->n, s->vs, g);
            if (m > 0) {
                if (s->emit && s->classes < s->emit_cap) {
                    memcpy(s->emit + s->classes * (long long)s->n * s->n, g, sizeof(int) * s->n * s->n);
                    s->mult_out[s->classes] = m;
                }
                s->classes++;
            }
            return;
        }
        if (s->emit) emit_grid(s);
        else if (s->emit_depth >= 0) s->emitted++;
        return;
    }
    int cell = s->order[step];
    int i = cell / s->n, j = cell % s->n, v;
    for (v = 0; v < s->n; v++) {
        if (!place(s, i, j, v)) continue;
        s->nodes++;
        if (s->level_nodes) s->level_nodes[step]++;
        fill(s, step + 1);
        unplace(s, i, j);
    }
}

static int load(oracle_state *s, int n, int vs, const int *grid, const int *order, int n_order)
{
    int i, j;
    if (n < 1 || n > MAXN) return -1;
    memset(s, 0, sizeof(*s));
    s->n = n; s->vs = vs; s->order = order; s->n_order = n_order; s->emit_depth = -1;
    for (i = 0; i < n; i++)
        for (j = 0; j < n; j++) s->ls[i][j] = grid ? grid[i * n + j] : -1;
    /* the given cells must themselves be consistent, else there is nothing to count */
    for (i = 0; i < n; i++)
        for (j = 0; j < n; j++) {
            int v = s->ls[i][j];
            if (v == -1) continue;
            if (v < 0 || v >= n) return -2;
            if (clashes(s, i, j, v)) return -2;
            if (vs && s->ls[i][n - 1 - j] != -1 && s->ls[i][n - 1 - j] != n - 1 - v) return -2;
        }
    for (i = 0; i < n_order; i++) {
        int c = order[i];
        if (c < 0 || c >= n * n || s->ls[c / n][c % n] != -1) return -3;
    }
    return 0;
}

/* Number of completions of `grid` (n*n ints, -1 empty) obtained by assigning the
 * cells of `order` (n_order cells, i*n+j) in that order.  `nodes` = number of
 * successful assignments made (every consistent partial square visited below
 * the root, leaves included).  Returns 0, or <0 on bad input. */
int oracle_count(int n, int vs, const int *grid, const int *order, int n_order,
                 unsigned long long *count, unsigned long long *nodes)
{
    oracle_state *s = (oracle_state *)malloc(sizeof(oracle_state));
    int rc = load(s, n, vs, grid, order, n_order);
    if (rc == 0) fill(s, 0);
    if (count) *count = rc == 0 ? s->count : 0;
    if (nodes) *nodes = rc == 0 ? s->nodes : 0;
    free(s);
    return rc;
}

/* oracle_count with the nodes split by depth: level_nodes[k] (k < n_order) =
 * number of successful assignments of order[k], i.e. of consistent partial
 * squares that assign exactly the first k+1 cells of the order (R9:
 * a node is one successful assignment).  Summing level_nodes[0..d-1] gives the
 * nodes of the search truncated after d cells (R15). */
int oracle_count_levels(int n, int vs, const int *grid, const int *order, int n_order,
                        unsigned long long *count, unsigned long long *level_nodes)
{
    oracle_state *s = (oracle_state *)malloc(sizeof(oracle_state));
    int rc = load(s, n, vs, grid, order, n_order), k;
    for (k = 0; k < n_order; k++) level_nodes[k] = 0;
    s->level_nodes = level_nodes;
    if (rc == 0) fill(s, 0);
    if (count) *count = rc == 0 ? s->count : 0;
    if (rc != 0)
        for (k = 0; k < n_order; k++) level_nodes[k] = 0;
    free(s);
    return rc;
}

/* All consistent assignments of the first `depth` cells of `order` (prefixes,
 * P:481).  Writes up to `cap` grids into out (n*n ints each, -1 for cells
 * outside the prefix) and returns the total number (which may exceed cap), or
 * <0 on bad input.  out may be NULL to just count. */
long long oracle_prefixes(int n, int vs, const int *grid, const int *order, int depth,
                          int *out, long long cap)
{
    oracle_state *s = (oracle_state *)malloc(sizeof(oracle_state));
    long long total;
    int rc = load(s, n, vs, grid, order, depth);
    if (rc != 0) { free(s); return rc; }
    s->emit = out; s->emit_cap = out ? cap : 0; s->emit_depth = depth;
    fill(s, 0);
    total = s->emitted;
    free(s);
    return total;
}

/* Every completion, written as full grids (up to cap); returns the number. */
long long oracle_squares(int n, int vs, const int *grid, const int *order, int n_order,
                         int *out, long long cap)
{
    oracle_state *s = (oracle_state *)malloc(sizeof(oracle_state));
    long long total;
    int rc = load(s, n, vs, grid, order, n_order);
    if (rc != 0) { free(s); return rc; }
    s->emit = out; s->emit_cap = out ? cap : 0;
    fill(s, 0);
    total = s->count;
    free(s);
    return total;
}

/* ------------------------------------------------------------------------ */
/* Cell order of Section 2.3.                                     */
/*                                                                            */
/* Only *which* cells are assigned matters, never their values.  At    */
/* each step:                                                                 */
/*  (forced) if some unit -- scanned rows 0..N-1, then columns 0..N-1,  */
/*     then the main diagonal, then the main antidiagonal -- has exactly N-1   */
/*     assigned cells, its remaining cell is taken next;                       */
/*  (V-score) otherwise take the unassigned cell with the largest       */
/*     V = r_i + c_j + md(i,j) + ad(i,j), the first in lexicographic (i,j)     */
/*     order among equal V.                                                    */
/* For vs (reading R4) the candidates are the left-half cells        */
/* (j <= N-1-j); taking (i,j) also marks (i,N-1-j) assigned, and a forced unit */
/* whose remaining cell is in the right half yields that cell's mirror.        */
/* `pre` marks cells assigned a priori (e.g. the fixed first row).      */
/* Returns the number of cells written to `order`.                            */
/* ------------------------------------------------------------------------ */
static int count_row(const int *a, int n, int i) { int k, c = 0; for (k = 0; k < n; k++) c += a[i * n + k]; return c; }
static int count_col(const int *a, int n, int j) { int k, c = 0; for (k = 0; k < n; k++) c += a[k * n + j]; return c; }
static int count_md(const int *a, int n) { int k, c = 0; for (k = 0; k < n; k++) c += a[k * n + k]; return c; }
static int count_ad(const int *a, int n) { int k, c = 0; for (k = 0; k < n; k++) c += a[k * n + (n - 1 - k)]; return c; }

int oracle_plan(int n, int vs, const int *pre, int *order)
{
    int a[MAXN * MAXN];
    int steps = 0, i, j, k;
    if (n < 1 || n > MAXN) return -1;
    for (k = 0; k < n * n; k++) a[k] = pre ? (pre[k] != 0) : 0;
    for (;;) {
        int pick = -1;
        /* forced cell: first unit (rows, columns, md, ad) with N-1 assigned */
        for (i = 0; i < n && pick < 0; i++)
            if (count_row(a, n, i) == n - 1)
                for (k = 0; k < n; k++) if (!a[i * n + k]) { pick = i * n + k; break; }
        for (j = 0; j < n && pick < 0; j++)
            if (count_col(a, n, j) == n - 1)
                for (k = 0; k < n; k++) if (!a[k * n + j]) { pick = k * n + j; break; }
        if (pick < 0 && count_md(a, n) == n - 1)
            for (k = 0; k < n; k++) if (!a[k * n + k]) { pick = k * n + k; break; }
        if (pick < 0 && count_ad(a, n) == n - 1)
            for (k = 0; k < n; k++) if (!a[k * n + n - 1 - k]) { pick = k * n + n - 1 - k; break; }
        if (pick < 0) {
            int best = -1;
            for (i = 0; i < n; i++)
                for (j = 0; j < n; j++) {
                    int v;
                    if (a[i * n + j]) continue;
                    if (vs && j > n - 1 - j) continue;
                    v = count_row(a, n, i) + count_col(a, n, j);
                    if (i == j) v += count_md(a, n);
                    if (i + j == n - 1) v += count_ad(a, n);
                    if (v > best) { best = v; pick = i * n + j; }
                }
        }
        if (pick < 0) break;                       /* everything assigned */
        if (vs) {
            int pi = pick / n, pj = pick % n;
            if (pj > n - 1 - pj) { pj = n - 1 - pj; pick = pi * n + pj; }
            a[pi * n + (n - 1 - pj)] = 1;
        }
        a[pick] = 1;
        order[steps++] = pick;
    }
    return steps;
}

/* ------------------------------------------------------------------------ */
/* M-transformations and canonisation of hourglass designs (Section 4,       */
/* P:297-438, Alg. 5).                                                       */
/*                                                                            */
/* An index map sigma acts on rows and columns alike: the pairs {k, N-1-k}   */
/* (k < h = floor(N/2)) are permuted by a permutation pi of 0..h-1 with      */
/* pi(0) = 0 (third type: row 0 may only meet row N-1), then the pairs */
/* in the subset `swap` have their two members exchanged (second type);*/
/* for odd N the middle index stays.  Optionally columns are then mirrored    */
/* (first type, vertical mirror; with symmetric pair swaps it also     */
/* yields the horizontal mirror).  The image is renamed so that row 0 reads  */
/* 0..N-1, empty cells stay empty.                            */
/* ------------------------------------------------------------------------ */

static void apply_m(int n, const int *g, const int *pi, int swap, int mirror, int *out)
{
    int sigma[MAXN], i, j, h = n / 2;
    int ren[MAXN];
    for (i = 0; i < n; i++) sigma[i] = i;
    for (i = 0; i < h; i++) {            /* pair i -> pair pi[i], then optional swap */
        int a = pi[i], lo = a, hi = n - 1 - a;
        if (swap & (1 << a)) { int t = lo; lo = hi; hi = t; }
        sigma[i] = lo;
        sigma[n - 1 - i] = hi;
    }
    for (i = 0; i < n * n; i++) out[i] = -1;
    for (i = 0; i < n; i++)
        for (j = 0; j < n; j++) {
            int v = g[i * n + j];
            int ti = sigma[i], tj = sigma[j];
            if (mirror) tj = n - 1 - tj;
            out[ti * n + tj] = v;
        }
    /* rename symbols so that row 0 is 0..N-1 (row 0 of an image is a full row) */
    for (j = 0; j < n; j++) ren[j] = -1;
    for (j = 0; j < n; j++) if (out[j] >= 0) ren[out[j]] = j;
    for (i = 0; i < n * n; i++) if (out[i] >= 0) out[i] = ren[out[i]];
}

static int lex_cmp(int n, const int *a, const int *b)
{
    int k;
    for (k = 0; k < n * n; k++) {
        if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
    }
    return 0;
}

static int next_perm(int *a, int m)      /* next lexicographic permutation of a[1..m-1] */
{
    int i = m - 2, j, t;
    while (i >= 1 && a[i] >= a[i + 1]) i--;
    if (i < 1) return 0;
    j = m - 1;
    while (a[j] <= a[i]) j--;
    t = a[i]; a[i] = a[j]; a[j] = t;
    for (i = i + 1, j = m - 1; i < j; i++, j--) { t = a[i]; a[i] = a[j]; a[j] = t; }
    return 1;
}

/* Alg. 5: 0 if some image is lexicographically smaller than g (g is
 * not the canonic form), else the number of distinct images (the power of its
 * class).  g must be normalised (row 0 = 0..N-1).  vs != 0: the vertical mirror
 * is left out (it is neutralised by vertical symmetry). */
long long oracle_canonize(int n, int vs, const int *g)
{
    int h = n / 2, pi[MAXN], swap, mirror, k;
    int (*imgs)[MAXN * MAXN];
    long long count = 0, distinct = 0, cap = 2LL << 5;
    {
        long long f = 1;
        for (k = 2; k < h; k++) f *= k;
        cap = 2LL * (1LL << h) * f;
    }
    imgs = malloc(sizeof(*imgs) * (size_t)cap);
    for (k = 0; k < h; k++) pi[k] = k;
    do {
        for (swap = 0; swap < (1 << h); swap++)
            for (mirror = 0; mirror < (vs ? 1 : 2); mirror++) {
                int t[MAXN * MAXN], c, seen = 0;
                long long e;
                apply_m(n, g, pi, swap, mirror, t);
                c = lex_cmp(n, t, g);
                if (c < 0) { free(imgs); return 0; }
                for (e = 0; e < count && !seen; e++) seen = lex_cmp(n, t, imgs[e]) == 0;
                if (!seen) { memcpy(imgs[count], t, sizeof(int) * n * n); count++; distinct++; }
            }
    } while (next_perm(pi, h));
    free(imgs);
    return distinct;
}

/* Alg. 6, first half: enumerate every design given by the first
 * `depth` cells of `order` below `grid` (the hourglass designs when `order` lists
 * the diagonals and row N-1), keep the canonic ones (Alg. 5) with their class
 * sizes.  Returns the number of classes (reps/mult written up to cap); *n_designs
 * receives the number of designs enumerated. */
long long oracle_classes(int n, int vs, const int *grid, const int *order, int depth,
                         int *reps, long long *mult, long long cap, long long *n_designs)
{
    oracle_state *s = (oracle_state *)malloc(sizeof(oracle_state));
    long long classes;
    int rc = load(s, n, vs, grid, order, depth);
    if (rc != 0) { free(s); return rc; }
    s->emit = reps; s->emit_cap = reps ? cap : 0; s->emit_depth = depth;
    s->canon = 1; s->mult_out = mult;
    fill(s, 0);
    classes = s->classes;
    if (n_designs) *n_designs = (long long)s->count;
    free(s);
    return classes;
}

/* One M-transformation (see apply_m) of a design, exported for the Proposition 1
 * tests: pi = permutation of the h pairs (pi[0] = 0), swap = subset of pairs. */
void oracle_transform(int n, const int *g, const int *pi, int swap, int mirror, int *out)
{
    apply_m(n, g, pi, swap, mirror, out);
}
