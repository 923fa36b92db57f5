/*
 * oracle/gbla_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the
 * Faugere-Lachartre reduction over GF(p) (arXiv 1602.06097, "GBLA").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, table or constant with the
 * CUDA path (paper_1602_06097_b200/csrc); neither includes the other.
 *
 * Every function cites the passage it follows ("P:n" = PAPER.md line n,
 * "S:n" = SPEC.md line n).  Readings of silent/garbled passages are the ones
 * listed in DESIGN.md §"Readings" (numbers R1..R22 = SURVEY.md §8(c) rows).
 *
 * Arithmetic: exact integers, least non-negative residues mod p; per-target
 * accumulators are uint64 and are reduced when a scalar is read and at
 * output (bound: n_piv * (p-1)^2 + p < 2^64 for n_piv < 2^32).
 *
 * Pinned by tests/test_oracle_pins.py (paper's multiline example P:524-556,
 * brute-force dense Gauss-Jordan over M*sigma on small inputs, closed forms
 * A*B' = B and C'*A = C, rank(M) = n_piv + rank(D_new), RREF idempotence and
 * row-permutation invariance, SPEC worked examples).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_NONE 0xFFFFFFFFu

/* ------------------------------------------------------------ field */

/* Trial division: p prime. */
int orc_is_prime(uint32_t p)
{
    if (p < 2) return 0;
    for (uint32_t d = 2; (uint64_t)d * d <= p; d++)
        if (p % d == 0) return 0;
    return 1;
}

/* Inverse by the extended Euclidean algorithm (reading R21).
 * Returns 0 for a == 0 (no inverse). */
uint32_t orc_inv(uint32_t a, uint32_t p)
{
    int64_t t = 0, newt = 1, r = p, newr = a % p;
    if (newr == 0) return 0;
    while (newr != 0) {
        int64_t q = r / newr, tmp;
        tmp = t - q * newt; t = newt; newt = tmp;
        tmp = r - q * newr; r = newr; newr = tmp;
    }
    if (r != 1) return 0;
    if (t < 0) t += p;
    return (uint32_t)t;
}

static inline uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p)
{
    return (uint32_t)(((uint64_t)a * b) % p);
}

/* ------------------------------------------------------------ validation */

/* O1: p prime with 2 < p < 2^16; CSR well-formed; columns strictly
 * increasing; values in [1, p).  0 = ok. */
int orc_validate(int64_t m, int64_t n, const uint64_t *row_ptr, const uint32_t *col,
                 const uint16_t *val, uint32_t p)
{
    if (p <= 2 || p >= 65536 || !orc_is_prime(p)) return 1;
    if (m < 0 || n < 0 || row_ptr[0] != 0) return 2;
    for (int64_t i = 0; i < m; i++) {
        if (row_ptr[i + 1] < row_ptr[i]) return 2;
        for (uint64_t q = row_ptr[i]; q < row_ptr[i + 1]; q++) {
            if ((int64_t)col[q] >= n) return 3;
            if (q > row_ptr[i] && col[q] <= col[q - 1]) return 3;
            if (val[q] == 0 || val[q] >= p) return 4;
        }
    }
    return 0;
}

/* ------------------------------------------------------------ Step 1: splice */

/*
 * Step 1.  Definitions used (readings R1-R7):
 *   lead(r)   = column of the first nonzero of row r (ORC_NONE for a zero row);
 *   weight(r) = number of nonzeros of r;
 *   P         = { lead(r) } (R2);
 *   pivot row of c in P = argmin (weight, row id) over rows with lead c (R1);
 *   sigma     = P ascending -> 0..npiv-1, then the other columns ascending ->
 *               npiv..n-1 (R3, R4);
 *   pivot rows in sigma(lead) order give A|B; all other rows (zero rows
 *   included) in original order give C|D (R5, R7).
 * Outputs: lead[m], sigma[n], pivot_row[npiv], nonpivot_row[mN]; returns 0.
 */
int orc_splice(int64_t m, int64_t n, const uint64_t *row_ptr, const uint32_t *col,
               uint32_t *lead, uint32_t *sigma, uint32_t *pivot_row, uint32_t *nonpivot_row,
               int64_t *npiv_out, int64_t *mN_out)
{
    int64_t *best = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t c = 0; c < n; c++) best[c] = -1;
    for (int64_t r = 0; r < m; r++) {
        uint64_t s = row_ptr[r], e = row_ptr[r + 1];
        if (s == e) { lead[r] = ORC_NONE; continue; }
        uint32_t c = col[s];
        lead[r] = c;
        int64_t b = best[c];
        if (b < 0) { best[c] = r; continue; }
        uint64_t wb = row_ptr[b + 1] - row_ptr[b], wr = e - s;
        if (wr < wb || (wr == wb && r < b)) best[c] = r;
    }
    int64_t npiv = 0;
    for (int64_t c = 0; c < n; c++) if (best[c] >= 0) npiv++;
    int64_t ip = 0, in = npiv;
    for (int64_t c = 0; c < n; c++) {
        if (best[c] >= 0) { pivot_row[ip] = (uint32_t)best[c]; sigma[c] = (uint32_t)ip++; }
        else sigma[c] = (uint32_t)in++;
    }
    int64_t mN = 0;
    for (int64_t r = 0; r < m; r++) {
        int is_piv = lead[r] != ORC_NONE && best[lead[r]] == r;
        if (!is_piv) nonpivot_row[mN++] = (uint32_t)r;
    }
    free(best);
    *npiv_out = npiv;
    *mN_out = mN;
    return 0;
}

/* Normalized row r scattered into the dense sigma-ordered vector `out`
 * (length n, residues): every nonzero row is multiplied by the inverse of
 * its leading value ("each polynomial is monic"; reading R6,
 * S:241-249). */
static void dense_normalized_row(int64_t r, const uint64_t *row_ptr, const uint32_t *col,
                                 const uint16_t *val, uint32_t p, const uint32_t *sigma,
                                 uint64_t *out)
{
    uint64_t s = row_ptr[r], e = row_ptr[r + 1];
    if (s == e) return;
    uint32_t il = orc_inv(val[s], p);
    for (uint64_t q = s; q < e; q++) out[sigma[col[q]]] = mulmod(val[q], il, p);
}

/* Dense quadrants in sigma order (small inputs only):
 * A npiv x npiv, B npiv x nN, C mN x npiv, D mN x nN, row-major uint32.
 * Any output pointer may be NULL. */
int orc_quadrants(int64_t m, int64_t n, const uint64_t *row_ptr, const uint32_t *col,
                  const uint16_t *val, uint32_t p, const uint32_t *sigma,
                  const uint32_t *pivot_row, int64_t npiv, const uint32_t *nonpivot_row, int64_t mN,
                  uint32_t *A, uint32_t *B, uint32_t *C, uint32_t *D)
{
    (void)m;
    int64_t nN = n - npiv;
    uint64_t *row = (uint64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint64_t));
    for (int64_t i = 0; i < npiv; i++) {
        memset(row, 0, (size_t)n * sizeof(uint64_t));
        dense_normalized_row(pivot_row[i], row_ptr, col, val, p, sigma, row);
        for (int64_t j = 0; j < npiv; j++) if (A) A[i * npiv + j] = (uint32_t)row[j];
        for (int64_t j = 0; j < nN; j++) if (B) B[i * nN + j] = (uint32_t)row[npiv + j];
    }
    for (int64_t i = 0; i < mN; i++) {
        memset(row, 0, (size_t)n * sizeof(uint64_t));
        dense_normalized_row(nonpivot_row[i], row_ptr, col, val, p, sigma, row);
        for (int64_t j = 0; j < npiv; j++) if (C) C[i * npiv + j] = (uint32_t)row[j];
        for (int64_t j = 0; j < nN; j++) if (D) D[i * nN + j] = (uint32_t)row[npiv + j];
    }
    free(row);
    return 0;
}

/* ------------------------------------------------ Alg 2: new order */

typedef struct {
    int64_t m, n, npiv, mN;
    const uint64_t *row_ptr; const uint32_t *col; const uint16_t *val; uint32_t p;
    const uint32_t *sigma, *pivot_row, *nonpivot_row;
    const int64_t *targets; int64_t ntargets;
    uint16_t *dnew; uint16_t *xout; uint64_t *modmac;
    int64_t next; pthread_mutex_t mu;
} dnew_job;

/*
 * Algorithm 2 "Reduction of C and D" for one target row t
 * (row t of C|D), read with R8 (subtract), R9 (the scalar dense_C[j] is
 * captured once, before both AXPYs, because A_jj = 1 zeroes it):
 *   dense = [C[t,*] | D[t,*]]                       (lines 660-661)
 *   for j = 0 .. npiv-1:                            (line 662)
 *     lambda = dense[j] mod p                       (line 663)
 *     if lambda != 0:
 *        dense -= lambda * [A[j,*] | B[j,*]]        (lines 664-665)
 *   D_new[t,*] = dense[npiv..] mod p                (line 668)
 * x_t[j] = lambda is row t of C' = C*A^-1 ("store the coefficients").
 * modMAC count: for every applied row, nnz(row_j) - 1 (the diagonal 1 only
 * cancels lambda).
 */
static void dnew_one(dnew_job *J, int64_t ti, uint64_t *acc)
{
    const int64_t n = J->n, npiv = J->npiv, nN = n - npiv;
    const uint32_t p = J->p;
    int64_t t = J->targets[ti];
    memset(acc, 0, (size_t)n * sizeof(uint64_t));
    dense_normalized_row(J->nonpivot_row[t], J->row_ptr, J->col, J->val, p, J->sigma, acc);
    uint64_t ops = 0;
    for (int64_t j = 0; j < npiv; j++) {
        uint32_t lambda = (uint32_t)(acc[j] % p);
        if (J->xout) J->xout[ti * npiv + j] = (uint16_t)lambda;
        if (lambda == 0) continue;
        uint32_t neg = p - lambda;
        int64_t r = J->pivot_row[j];
        uint64_t s = J->row_ptr[r], e = J->row_ptr[r + 1];
        uint32_t il = orc_inv(J->val[s], p);
        for (uint64_t q = s; q < e; q++) {
            uint32_t v = mulmod(J->val[q], il, p);
            acc[J->sigma[J->col[q]]] += (uint64_t)neg * v;
        }
        ops += (e - s) - 1;
    }
    for (int64_t k = 0; k < nN; k++) J->dnew[ti * nN + k] = (uint16_t)(acc[npiv + k] % p);
    if (J->modmac) J->modmac[ti] = ops;
}

static void *dnew_worker(void *arg)
{
    dnew_job *J = (dnew_job *)arg;
    uint64_t *acc = (uint64_t *)malloc((size_t)(J->n > 0 ? J->n : 1) * sizeof(uint64_t));
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t ti = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (ti >= J->ntargets) break;
        dnew_one(J, ti, acc);
    }
    free(acc);
    return NULL;
}

/* D_new rows (and optionally C' rows and modMAC counts) for a list of
 * targets (indices into the non-pivot rows).  dnew: ntargets x nN;
 * xout: ntargets x npiv or NULL; modmac: ntargets or NULL.
 * Threads only split the independent targets. */
int orc_dnew(int64_t m, int64_t n, const uint64_t *row_ptr, const uint32_t *col,
             const uint16_t *val, uint32_t p, const uint32_t *sigma,
             const uint32_t *pivot_row, int64_t npiv, const uint32_t *nonpivot_row, int64_t mN,
             const int64_t *targets, int64_t ntargets,
             uint16_t *dnew, uint16_t *xout, uint64_t *modmac, int threads)
{
    dnew_job J = { m, n, npiv, mN, row_ptr, col, val, p, sigma, pivot_row, nonpivot_row,
                   targets, ntargets, dnew, xout, modmac, 0, PTHREAD_MUTEX_INITIALIZER };
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    for (int i = 0; i < threads; i++) pthread_create(&th[i], NULL, dnew_worker, &J);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    return 0;
}

/* ------------------------------------------- Step 2 and Step 3, standard order */

/*
 * Step 2, TRSM: B' = A^-1 B with A upper unitriangular, by
 * back substitution, rows i = npiv-1 .. 0:
 *   B'_i = B_i - sum_{j > i, A_ij != 0} A_ij * B'_j.
 * Dense A (npiv x npiv), B and Bp (npiv x nN), residues.
 */
int orc_trsm(const uint32_t *A, const uint32_t *B, uint32_t *Bp, int64_t npiv, int64_t nN, uint32_t p)
{
    uint64_t *acc = (uint64_t *)malloc((size_t)(nN > 0 ? nN : 1) * sizeof(uint64_t));
    for (int64_t i = npiv - 1; i >= 0; i--) {
        for (int64_t k = 0; k < nN; k++) acc[k] = B[i * nN + k];
        for (int64_t j = i + 1; j < npiv; j++) {
            uint32_t a = A[i * npiv + j];
            if (!a) continue;
            for (int64_t k = 0; k < nN; k++) acc[k] = (acc[k] + (uint64_t)(p - a) * Bp[j * nN + k]) % p;
        }
        for (int64_t k = 0; k < nN; k++) Bp[i * nN + k] = (uint32_t)(acc[k] % p);
    }
    free(acc);
    return 0;
}

/* Step 3 and the 4-step variant's last step:
 * Dout = D - X * Y  (X: rows x inner, Y: inner x cols, residues).
 * Standard order: X = C, Y = B' ; new order: X = C', Y = B. */
int orc_sub_mul(const uint32_t *D, const uint32_t *X, const uint32_t *Y, uint32_t *Dout,
                int64_t rows, int64_t inner, int64_t cols, uint32_t p)
{
    for (int64_t i = 0; i < rows; i++)
        for (int64_t k = 0; k < cols; k++) {
            uint64_t s = 0;
            for (int64_t j = 0; j < inner; j++) s = (s + (uint64_t)X[i * inner + j] * Y[j * cols + k]) % p;
            Dout[i * cols + k] = (uint32_t)((D[i * cols + k] + p - s) % p);
        }
    return 0;
}

/* ----------------------------------------------------- Step 4: RREF of D_new */

typedef struct {
    uint32_t *a; int64_t rows, cols; uint32_t p; int threads;
    pthread_barrier_t bar;
    volatile int64_t piv_row; volatile int64_t col; volatile int done;
} rref_job;

typedef struct { rref_job *J; int id; } rref_arg;

/* Worker: eliminate column J->col from every row except J->piv_row, using the
 * (already normalized) pivot row; rows are split among threads. */
static void *rref_worker(void *arg)
{
    rref_arg *A = (rref_arg *)arg;
    rref_job *J = A->J;
    for (;;) {
        pthread_barrier_wait(&J->bar);           /* a column is ready (or done) */
        if (J->done) break;
        int64_t c = J->col, pr = J->piv_row, cols = J->cols;
        uint32_t p = J->p;
        const uint32_t *prow = J->a + pr * cols;
        for (int64_t i = A->id; i < J->rows; i += J->threads) {
            if (i == pr) continue;
            uint32_t *row = J->a + i * cols;
            uint32_t f = row[c];
            if (!f) continue;
            uint32_t nf = p - f;
            for (int64_t k = c; k < cols; k++)
                row[k] = (uint32_t)((row[k] + (uint64_t)nf * prow[k]) % p);
        }
        pthread_barrier_wait(&J->bar);           /* column finished */
    }
    return NULL;
}

/*
 * Canonical reduced row echelon form (reading R13):
 * Gauss-Jordan column by column: for each column c, the first not-yet-used
 * row with a nonzero at c becomes the pivot; it is swapped into position r,
 * scaled by the inverse of its entry, and column c is eliminated from ALL
 * other rows; r++.  On return rows 0..rank-1 hold R, pivcol[0..rank-1] the
 * pivot columns; the remaining rows are zero.  Matrix: rows x cols, residues.
 */
int64_t orc_rref(uint32_t *a, int64_t rows, int64_t cols, uint32_t p, uint32_t *pivcol, int threads)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    rref_job J;
    J.a = a; J.rows = rows; J.cols = cols; J.p = p; J.threads = threads; J.done = 0;
    pthread_barrier_init(&J.bar, NULL, (unsigned)threads + 1);
    pthread_t th[256];
    rref_arg args[256];
    for (int i = 0; i < threads; i++) { args[i].J = &J; args[i].id = i; pthread_create(&th[i], NULL, rref_worker, &args[i]); }
    int64_t r = 0;
    uint32_t *tmp = (uint32_t *)malloc((size_t)(cols > 0 ? cols : 1) * sizeof(uint32_t));
    for (int64_t c = 0; c < cols && r < rows; c++) {
        int64_t s = -1;
        for (int64_t i = r; i < rows; i++) if (a[i * cols + c]) { s = i; break; }
        if (s < 0) continue;
        if (s != r) {
            memcpy(tmp, a + s * cols, (size_t)cols * sizeof(uint32_t));
            memcpy(a + s * cols, a + r * cols, (size_t)cols * sizeof(uint32_t));
            memcpy(a + r * cols, tmp, (size_t)cols * sizeof(uint32_t));
        }
        uint32_t inv = orc_inv(a[r * cols + c], p);
        for (int64_t k = c; k < cols; k++) a[r * cols + k] = mulmod(a[r * cols + k], inv, p);
        J.col = c; J.piv_row = r;
        pthread_barrier_wait(&J.bar);   /* release workers */
        pthread_barrier_wait(&J.bar);   /* wait for them */
        pivcol[r] = (uint32_t)c;
        r++;
    }
    J.done = 1;
    pthread_barrier_wait(&J.bar);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    pthread_barrier_destroy(&J.bar);
    free(tmp);
    return r;
}

/* ------------------------------------------------------- multiline */

/*
 * 2-multiline vector of two sparse rows given densely (Definition):
 * pos = columns where at least one of the two rows is nonzero (ascending);
 * val[2i], val[2i+1] = the two rows' entries at pos[i] (zeros allowed).
 * Returns the length l; pos has room for len entries, val for 2*len.
 */
int64_t orc_multiline(const uint32_t *r1, const uint32_t *r2, int64_t len, uint32_t *pos, uint32_t *val)
{
    int64_t l = 0;
    for (int64_t c = 0; c < len; c++) {
        if (r1[c] == 0 && r2[c] == 0) continue;
        pos[l] = (uint32_t)c;
        val[2 * l] = r1[c];
        val[2 * l + 1] = r2[c];
        l++;
    }
    return l;
}

/*
 * Algorithm 1 read with reading R10 (subtract; the assignment
 * "dense_1[k] <- lambda11 v1 + lambda12 v2" is an update):
 *   dense1[pos[i]] -= l11*val[2i] + l12*val[2i+1]
 *   dense2[pos[i]] -= l21*val[2i] + l22*val[2i+1]
 * dense rows are residues, updated in place.
 */
void orc_ml_axpy(uint32_t *d1, uint32_t *d2, uint32_t l11, uint32_t l12, uint32_t l21, uint32_t l22,
                 const uint32_t *pos, const uint32_t *val, int64_t l, uint32_t p)
{
    for (int64_t i = 0; i < l; i++) {
        uint32_t k = pos[i];
        uint64_t v1 = val[2 * i], v2 = val[2 * i + 1];
        uint64_t s1 = ((uint64_t)l11 * v1 + (uint64_t)l12 * v2) % p;
        uint64_t s2 = ((uint64_t)l21 * v1 + (uint64_t)l22 * v2) % p;
        d1[k] = (uint32_t)((d1[k] + p - s1) % p);
        d2[k] = (uint32_t)((d2[k] + p - s2) % p);
    }
}
