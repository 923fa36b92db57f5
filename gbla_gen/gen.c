/*
 * gbla_gen/gen.c -- seeded synthetic input generator (shared by the oracle
 * and the CUDA path; holds NONE of the method's arithmetic).
 *
 * Produces F4/F5-shaped Macaulay matrices over GF(p) in CSR form
 * (row_ptr u64[m+1], col u32[nnz] strictly increasing per row,
 *  val u16[nnz] in [1, p-1]) following the recipe of SURVEY.md §8(d)
 * G1-G8 and DESIGN.md "Input recipe":
 *   - near-triangular structure with pivot columns (PAPER.md P:61-66,
 *     P:359-371), horizontal runs and vertical pattern sharing,
 *     n_piv >> m - n_piv;
 *   - monic rows;
 *   - planted rank of D via dependent rows built as lambda1*r_a + lambda2*r_b
 *     with lambda1 + lambda2 = 1 when leads coincide (no inverse needed).
 * Also a plain random sparse matrix generator (non-monic, arbitrary leads,
 * zero rows) for the small randomized parity suite.
 *
 * PRNG: counter-based SplitMix64 keyed by (seed, stream, row) so that the
 * output is deterministic and independent of thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t m, n, npiv;       /* rows, columns, generator pivot rows            */
    int64_t rank_planted;     /* independent non-pivot rows                     */
    int64_t k;                /* target nonzeros per pivot row                  */
    int64_t run;              /* run length R                                   */
    int64_t band;             /* W for pivot rows (0 = up to the last column)   */
    int64_t band_np;          /* W for non-pivot rows (0 = up to last column)   */
    int64_t chain;            /* pattern-sharing chain restart period (rows)    */
    double share;             /* probability of inheriting a run of row i-1     */
    double lead_frac;         /* >0: non-pivot leads among pivots < lead_frac*n */
    uint32_t p;
    uint32_t pad_;
    uint64_t seed;
} gen_params;

typedef struct {
    int64_t m, n, nnz;
    uint64_t *row_ptr;
    uint32_t *col;
    uint16_t *val;
    uint32_t *piv;            /* generator pivot columns, sorted (npiv)       */
    int64_t npiv;
} gen_out;

/* ------------------------------------------------------------------ PRNG */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
typedef struct { uint64_t s; } rng_t;
static inline rng_t rng_for(uint64_t seed, uint64_t stream, uint64_t row) {
    rng_t r;
    r.s = mix64(seed * 0x9E3779B97F4A7C15ull + mix64(stream + 0x1234567ull) + mix64(row ^ 0xA5A5A5A5DEADBEEFull));
    return r;
}
static inline uint64_t rng_next(rng_t *r) {
    r->s += 0x9E3779B97F4A7C15ull;
    return mix64(r->s);
}
/* uniform in [0, bound), bound < 2^32 */
static inline uint64_t rng_below(rng_t *r, uint64_t bound) {
    return ((rng_next(r) >> 32) * bound) >> 32;
}
static inline double rng_unit(rng_t *r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }

/* ------------------------------------------------------- growable buffers */
typedef struct { uint32_t *c; uint16_t *v; int64_t len, cap; } rowbuf;
static void rb_push(rowbuf *b, uint32_t c, uint16_t v) {
    if (b->len == b->cap) {
        b->cap = b->cap ? b->cap * 2 : 1024;
        b->c = (uint32_t *)realloc(b->c, (size_t)b->cap * sizeof(uint32_t));
        b->v = (uint16_t *)realloc(b->v, (size_t)b->cap * sizeof(uint16_t));
    }
    b->c[b->len] = c; b->v[b->len] = v; b->len++;
}

typedef struct { uint32_t *a, *b; int64_t len, cap; } runlist;   /* [a, b) */
static void rl_push(runlist *l, uint32_t a, uint32_t b) {
    if (l->len == l->cap) {
        l->cap = l->cap ? l->cap * 2 : 64;
        l->a = (uint32_t *)realloc(l->a, (size_t)l->cap * sizeof(uint32_t));
        l->b = (uint32_t *)realloc(l->b, (size_t)l->cap * sizeof(uint32_t));
    }
    l->a[l->len] = a; l->b[l->len] = b; l->len++;
}

static int cmp_u32(const void *x, const void *y) {
    uint32_t a = *(const uint32_t *)x, b = *(const uint32_t *)y;
    return (a > b) - (a < b);
}

/* Fill runs of length `run` into the window [lo, hi] (inclusive) until `want`
 * columns are occupied.  `occ` is a byte map over [0, n) that is clean on
 * entry and clean on exit.  Inherited runs (from `prev`) are kept with
 * probability `share` first.  Result: sorted column list in `cols`. */
static void draw_runs(rng_t *r, uint8_t *occ, int64_t lo, int64_t hi, int64_t want,
                      int64_t run, const runlist *prev, double share, runlist *cur,
                      uint32_t *cols, int64_t *ncols)
{
    int64_t have = 0;
    cur->len = 0;
    if (hi < lo) { *ncols = 0; return; }
    int64_t span = hi - lo + 1;
    if (want > span) want = span;
    if (prev) {
        for (int64_t i = 0; i < prev->len && have < want; i++) {
            int64_t a = prev->a[i], b = prev->b[i];
            if (a < lo) continue;            /* only runs lying right of the lead */
            if (a > hi) continue;
            if (b > hi + 1) b = hi + 1;
            if (rng_unit(r) >= share) continue;
            if (b - a > want - have) b = a + (want - have);
            for (int64_t c = a; c < b; c++) occ[c] = 1;
            rl_push(cur, (uint32_t)a, (uint32_t)b);
            have += b - a;
        }
    }
    int64_t attempts = 0, max_attempts = 64 * (want / (run > 0 ? run : 1) + 8);
    while (have < want && attempts < max_attempts) {
        attempts++;
        int64_t nstart = span - run + 1;
        if (nstart < 1) nstart = 1;
        int64_t a = lo + (int64_t)rng_below(r, (uint64_t)nstart);
        int64_t b = a + run;
        if (b > hi + 1) b = hi + 1;
        if (b - a > want - have) b = a + (want - have);
        int ok = 1;
        for (int64_t c = a; c < b; c++) if (occ[c]) { ok = 0; break; }
        if (!ok) continue;
        for (int64_t c = a; c < b; c++) occ[c] = 1;
        rl_push(cur, (uint32_t)a, (uint32_t)b);
        have += b - a;
    }
    /* deterministic completion if rejection sampling stalled (dense windows) */
    for (int64_t c = lo; c <= hi && have < want; c++) {
        if (!occ[c]) { occ[c] = 1; rl_push(cur, (uint32_t)c, (uint32_t)(c + 1)); have++; }
    }
    int64_t nc = 0;
    for (int64_t i = 0; i < cur->len; i++)
        for (uint32_t c = cur->a[i]; c < cur->b[i]; c++) cols[nc++] = c;
    qsort(cols, (size_t)nc, sizeof(uint32_t), cmp_u32);
    for (int64_t i = 0; i < nc; i++) occ[cols[i]] = 0;
    *ncols = nc;
}

void gen_free(gen_out *o) {
    free(o->row_ptr); free(o->col); free(o->val); free(o->piv);
    memset(o, 0, sizeof(*o));
}

/* F4/F5-shaped matrix.  Returns 0 on success. */
int gen_f4(const gen_params *P, gen_out *out)
{
    memset(out, 0, sizeof(*out));
    const int64_t m = P->m, n = P->n, npiv = P->npiv, mN = m - npiv;
    const int64_t rho = P->rank_planted;
    const uint32_t p = P->p;
    if (npiv <= 0 || npiv > n || mN < 0 || rho > mN || rho < 1 || p < 3 || P->k < 1 || P->run < 1)
        return -1;

    /* G2: pivot columns = uniformly random sorted npiv-subset of [0, n)
     * (selection sampling, Knuth Algorithm S). */
    uint32_t *piv = (uint32_t *)malloc((size_t)npiv * sizeof(uint32_t));
    {
        rng_t r = rng_for(P->seed, 1, 0);
        int64_t need = npiv;
        for (int64_t c = 0, j = 0; c < n && need > 0; c++) {
            if ((int64_t)rng_below(&r, (uint64_t)(n - c)) < need) { piv[j++] = (uint32_t)c; need--; }
        }
    }

    rowbuf all = {0};                 /* concatenated rows, in generation order */
    int64_t *start = (int64_t *)malloc((size_t)(m + 1) * sizeof(int64_t));
    uint8_t *occ = (uint8_t *)calloc((size_t)n, 1);
    uint32_t *cols = (uint32_t *)malloc((size_t)(n + 1) * sizeof(uint32_t));
    runlist prev = {0}, cur = {0};
    int64_t row = 0;

    /* G3: pivot rows. */
    for (int64_t i = 0; i < npiv; i++, row++) {
        rng_t r = rng_for(P->seed, 2, (uint64_t)i);
        int64_t c0 = piv[i];
        int64_t hi = P->band > 0 ? c0 + P->band : n - 1;
        if (hi > n - 1) hi = n - 1;
        int64_t nc = 0;
        int inherit = (P->chain <= 0 || (i % P->chain) != 0) && i > 0;
        draw_runs(&r, occ, c0 + 1, hi, P->k - 1, P->run, inherit ? &prev : NULL, P->share,
                  &cur, cols, &nc);
        start[row] = all.len;
        rb_push(&all, (uint32_t)c0, 1);
        for (int64_t t = 0; t < nc; t++) rb_push(&all, cols[t], (uint16_t)(1 + rng_below(&r, p - 1)));
        runlist tmp = prev; prev = cur; cur = tmp;
    }

    /* G4: independent non-pivot rows (leads at pivot columns, heavier by one run). */
    int64_t elig = 0;
    for (int64_t i = 0; i < npiv; i++) {
        int ok;
        if (P->lead_frac > 0) ok = (double)piv[i] < P->lead_frac * (double)n;
        else if (P->band_np > 0) ok = piv[i] + P->band_np <= n - 1;
        else ok = piv[i] + 2 * (P->k + P->run) <= n - 1;
        if (ok) elig = i + 1; else if (P->lead_frac <= 0) break;
    }
    if (elig < 1) elig = 1;
    int64_t *indep_start = (int64_t *)malloc((size_t)(rho > 0 ? rho : 1) * sizeof(int64_t));
    for (int64_t t = 0; t < rho; t++, row++) {
        rng_t r = rng_for(P->seed, 3, (uint64_t)t);
        int64_t li = (int64_t)rng_below(&r, (uint64_t)elig);
        int64_t c0 = piv[li];
        int64_t hi = P->band_np > 0 ? c0 + P->band_np : n - 1;
        if (hi > n - 1) hi = n - 1;
        int64_t nc = 0;
        draw_runs(&r, occ, c0 + 1, hi, P->k - 1 + P->run, P->run, NULL, 0.0, &cur, cols, &nc);
        start[row] = all.len;
        indep_start[t] = row;
        rb_push(&all, (uint32_t)c0, 1);
        for (int64_t q = 0; q < nc; q++) rb_push(&all, cols[q], (uint16_t)(1 + rng_below(&r, p - 1)));
    }
    start[row] = all.len;   /* provisional end for the independent block */

    /* G5: dependent rows = l1*r_a + l2*r_b, monic by construction.
     * Rows are contiguous in generation order: row q is [start[q], start[q+1]). */
    int64_t ndep = mN - rho;
    for (int64_t t = 0; t < ndep; t++, row++) {
        rng_t r = rng_for(P->seed, 4, (uint64_t)t);
        int64_t a = (int64_t)rng_below(&r, (uint64_t)rho), b;
        if (rho < 2) b = a; else { do { b = (int64_t)rng_below(&r, (uint64_t)rho); } while (b == a); }
        int64_t ra = indep_start[a], rb = indep_start[b];
        uint32_t la = all.c[start[ra]], lb = all.c[start[rb]];
        uint64_t l1, l2;
        if (la < lb) { l1 = 1; l2 = 1 + rng_below(&r, p - 1); }
        else if (lb < la) { l2 = 1; l1 = 1 + rng_below(&r, p - 1); }
        else { l1 = 2 + rng_below(&r, p - 2); l2 = (1 + p - l1) % p; }   /* l1 + l2 = 1 */
        int64_t ia = start[ra], ea = start[ra + 1], ib = start[rb], eb = start[rb + 1];
        start[row] = all.len;
        while (ia < ea || ib < eb) {
            uint32_t ca = ia < ea ? all.c[ia] : UINT32_MAX;
            uint32_t cb = ib < eb ? all.c[ib] : UINT32_MAX;
            uint64_t v; uint32_t c;
            if (ca < cb) { c = ca; v = (l1 * all.v[ia]) % p; ia++; }
            else if (cb < ca) { c = cb; v = (l2 * all.v[ib]) % p; ib++; }
            else { c = ca; v = (l1 * all.v[ia] + l2 * all.v[ib]) % p; ia++; ib++; }
            if (v) rb_push(&all, c, (uint16_t)v);
        }
    }
    start[m] = all.len;

    /* G7: seeded random row order. */
    int64_t *perm = (int64_t *)malloc((size_t)m * sizeof(int64_t));
    for (int64_t q = 0; q < m; q++) perm[q] = q;
    {
        rng_t r = rng_for(P->seed, 7, 0);
        for (int64_t q = m - 1; q > 0; q--) {
            int64_t j = (int64_t)rng_below(&r, (uint64_t)(q + 1));
            int64_t tmp = perm[q]; perm[q] = perm[j]; perm[j] = tmp;
        }
    }
    int64_t nnz = all.len;
    out->m = m; out->n = n; out->nnz = nnz; out->npiv = npiv; out->piv = piv;
    out->row_ptr = (uint64_t *)malloc((size_t)(m + 1) * sizeof(uint64_t));
    out->col = (uint32_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(uint32_t));
    out->val = (uint16_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(uint16_t));
    uint64_t pos = 0;
    for (int64_t q = 0; q < m; q++) {
        int64_t src = perm[q];
        out->row_ptr[q] = pos;
        int64_t len = start[src + 1] - start[src];
        memcpy(out->col + pos, all.c + start[src], (size_t)len * sizeof(uint32_t));
        memcpy(out->val + pos, all.v + start[src], (size_t)len * sizeof(uint16_t));
        pos += (uint64_t)len;
    }
    out->row_ptr[m] = pos;

    free(perm); free(indep_start); free(start); free(occ); free(cols);
    free(prev.a); free(prev.b); free(cur.a); free(cur.b); free(all.c); free(all.v);
    return 0;
}

/* Plain random sparse matrix: each entry nonzero with probability `density`,
 * value uniform in [1, p-1]; rows are NOT normalized (exercises Step-1
 * normalization, ties and zero rows). */
int gen_random(int64_t m, int64_t n, double density, uint32_t p, uint64_t seed, gen_out *out)
{
    memset(out, 0, sizeof(*out));
    rowbuf all = {0};
    out->row_ptr = (uint64_t *)malloc((size_t)(m + 1) * sizeof(uint64_t));
    for (int64_t i = 0; i < m; i++) {
        rng_t r = rng_for(seed, 11, (uint64_t)i);
        out->row_ptr[i] = (uint64_t)all.len;
        for (int64_t c = 0; c < n; c++)
            if (rng_unit(&r) < density) rb_push(&all, (uint32_t)c, (uint16_t)(1 + rng_below(&r, p - 1)));
    }
    out->row_ptr[m] = (uint64_t)all.len;
    out->m = m; out->n = n; out->nnz = all.len;
    out->col = all.c ? all.c : (uint32_t *)malloc(4);
    out->val = all.v ? all.v : (uint16_t *)malloc(2);
    out->piv = NULL; out->npiv = 0;
    return 0;
}
