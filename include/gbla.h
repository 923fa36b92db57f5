/*
 * gbla.h -- C ABI of libgbla: Faugere-Lachartre reduction of F4/F5
 * Macaulay matrices over GF(p), p < 2^16, on NVIDIA B200 (sm_100a).
 *
 * Paper: Boyer, Eder, Faugere, Lachartre, Martani, "GBLA -- Groebner Basis
 * Linear Algebra Package", arXiv 1602.06097.  Citations "P:n" are lines of
 * its LaTeX source; DESIGN.md lists the readings R1..R22 of
 * passages the paper leaves silent or garbled.
 *
 * Conventions for every call
 *   - All matrix pointers are DEVICE pointers unless the GBLA_HOST_INPUT flag
 *     says otherwise.  Work is enqueued on `stream` (a cudaStream_t passed as
 *     void*, NULL = legacy default stream); calls that must learn sizes
 *     (gbla_splice, gbla_echelon_D) synchronize that stream.
 *   - Inputs are caller-owned and never written; they must stay valid until
 *     the stream work that reads them completes.  Every buffer the library
 *     creates is owned by the handle that created it and is released by
 *     gbla_mat_free / gbla_ctx_destroy.  Device memory comes from the
 *     context's allocator (gbla_ctx_set_allocator; default cudaMallocAsync).
 *   - All outputs are canonical residues in [0, p).
 *   - Errors: host-checkable problems (NULL pointers, sizes, p not a prime in
 *     (2, 2^16), unknown flags, call order) return a status synchronously
 *     and change nothing.  Input errors found on the device (unsorted or
 *     duplicate columns, col >= n, val == 0 or val >= p) are latched and
 *     returned as GBLA_E_INVAL by gbla_splice (which synchronizes); the
 *     handle is then not created.  gbla_last_error() gives a thread-local
 *     message for the last non-OK status.  There is no CPU fallback: without
 *     a usable sm_100 device every compute call returns GBLA_E_CUDA.
 *   - A gbla_mat handle is single-stream and single-thread.
 */
#ifndef GBLA_H
#define GBLA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GBLA_OK = 0,
    GBLA_E_INVAL = 1,    /* malformed input (pointers, sizes, CSR content)       */
    GBLA_E_DOMAIN = 2,   /* p not prime or not in (2, 2^16)                      */
    GBLA_E_ORDER = 3,    /* call sequence violates the contract below            */
    GBLA_E_NOMEM = 4,    /* device allocation failed                             */
    GBLA_E_CUDA = 5,     /* CUDA runtime error / no sm_100 device                */
    GBLA_E_NCCL = 6,     /* NCCL error (multi-GPU)                               */
    GBLA_E_INTERNAL = 7
} gbla_status;

/* ---- flags ------------------------------------------------------------ */
#define GBLA_ORDER_NEW       0x00u  /* gbla_reduce: new order, Alg 2 [default] */
#define GBLA_ORDER_STANDARD  0x01u  /* gbla_reduce: Steps 2-3 with TRSM        */
#define GBLA_FUSE_D          0x02u  /* gbla_reduce_C: also update D (Alg 2)  */
#define GBLA_HOST_INPUT      0x04u  /* gbla_splice/gbla_reduce: M's arrays are host memory */
#define GBLA_KEEP_CPRIME     0x08u  /* fused gbla_reduce_C also stores C' = C A^-1         */
#define GBLA_SPARSE_INT      0x10u  /* sparse phase: per-target multiline AXPY (INT pipe)  */
#define GBLA_DENSE_INT       0x20u  /* echelon trailing update on the INT pipe             */
#define GBLA_DENSE_TC        0x40u  /* echelon trailing update on tcgen05 (u8-limb IMMA)   */
#define GBLA_ECHELON_REF     0x80u  /* echelon_D: row echelon form only, no elimination
                                       above the pivots (rank / reduction-of-D use case of
                                       the F5 runs; Alg 3's non-reduced echelon,
                                       P:715-740)                          */
#define GBLA_FLAGS_ALL       0xFFu

/* ---- input ------------------------------------------------------------ */
/* Sparse matrix M (m x n) over GF(p) in CSR: row i holds the entries
 * (col[q], val[q]) for q in [row_ptr[i], row_ptr[i+1]); columns strictly
 * increasing within a row, 1 <= val < p.  Rows are polynomials, columns
 * monomials in decreasing monomial order.  Rows need not be
 * monic: Step 1 normalizes them (reading R6).  Zero rows are
 * allowed (reading R7).  m, n < 2^31. */
typedef struct {
    int64_t m, n, nnz;
    const uint64_t *row_ptr;   /* m+1 */
    const uint32_t *col;       /* nnz */
    const uint16_t *val;       /* nnz */
} gbla_csr;

typedef struct gbla_ctx_s *gbla_ctx;   /* device, allocator, optional NCCL comm */
typedef struct gbla_mat_s *gbla_mat;   /* one spliced matrix and its results    */

typedef void *(*gbla_alloc_fn)(size_t bytes, void *stream, void *user);
typedef void (*gbla_free_fn)(void *ptr, void *stream, void *user);

/* ---- context ---------------------------------------------------------- */
/* Bind to CUDA device `device` (must be sm_100).  GBLA_E_CUDA otherwise. */
gbla_status gbla_ctx_create(int device, gbla_ctx *out);
/* Route every device allocation through (alloc, free); NULL restores the
 * default (cudaMallocAsync / cudaFreeAsync on the call's stream). */
gbla_status gbla_ctx_set_allocator(gbla_ctx ctx, gbla_alloc_fn alloc, gbla_free_fn free_fn, void *user);
/* Optional: bytes the context's allocator can still provide (the driver's free memory plus what
 * a caching allocator holds unused).  The sparse phase sizes its batches of X tiles from it
 * (without it: cudaMemGetInfo, which does not see a caching allocator's free blocks).  fn is
 * called on the host thread that calls the library; NULL restores the default. */
typedef size_t (*gbla_memq_fn)(void *user);
gbla_status gbla_ctx_set_mem_query(gbla_ctx ctx, gbla_memq_fn fn, void *user);
/* Multi-GPU: join an NCCL communicator built from a 128-byte ncclUniqueId
 * shared by the caller (e.g. through torch.distributed), as `rank` of
 * `world`.  Collective: every rank must call it.  nccl_unique_id == NULL
 * (world 1) detaches; world == 1 WITH an id builds a one-rank communicator:
 * the distributed code path (C1 broadcast, sharded sparse phase, distributed
 * echelon) and every NCCL call in it then run on one GPU (tests).  Input
 * errors found by rank 0 are returned by every rank (they travel with the
 * C1 dims broadcast); asynchronous NCCL errors are polled
 * (ncclCommGetAsyncError) at every host wait of a distributed phase, abort the
 * communicator and return GBLA_E_NCCL. */
gbla_status gbla_ctx_set_comm(gbla_ctx ctx, const void *nccl_unique_id, int rank, int world);
/* Fill out128 with a fresh ncclUniqueId (call on one rank, broadcast it). */
gbla_status gbla_nccl_get_unique_id(void *out128);
void gbla_ctx_destroy(gbla_ctx ctx);

/* ---- the six calls (north star) ------------------------ */

/* Step 1: normalize rows; lead(r) = first column;
 * pivot columns P = { lead(r) } (R2); for each c in P the pivot row is the
 * candidate of minimum (weight, row id) (R1: "keep A as sparse as
 * possible"); sigma orders P ascending then the other columns
 * ascending (R3, R4); pivot rows in sigma(lead) order form A|B, all other
 * rows in original order form C|D (R5, R7).  Builds the device formats
 * (sigma-ordered rows and the dense D quadrant; the two-row multilines of
 * A|B, are built on first use: gbla_get_multilines or the
 * GBLA_SPARSE_INT path).  Synchronizes `stream`.  flags: GBLA_HOST_INPUT only. */
gbla_status gbla_splice(gbla_ctx ctx, const gbla_csr *M, uint32_t p, uint32_t flags,
                        void *stream, gbla_mat *out);

/* Step 2, TRSM: B <- A^-1 B (A unit upper triangular; "one only
 * reads A and writes to B").  Result kept as dense B' (n_piv x nN, u16
 * residues, row stride from gbla_get_Bprime), owned by h.  Default engine:
 * the tensor-core sparse phase applied to the unit targets e_k (row k of
 * -A^-1 B is the D_new row of the target e_k; exact), then negated;
 * environment GBLA_TRSM_INT=1 selects the INT-pipe back substitution (one
 * thread per column).  Synchronizes `stream`.  Errors: GBLA_E_ORDER if
 * already done, GBLA_E_NOMEM, GBLA_E_CUDA, GBLA_E_INTERNAL. */
gbla_status gbla_reduce_B(gbla_mat h, void *stream);

/* C <- C A^-1 (new order): per non-pivot row, forward
 * substitution over the pivots in ascending order, lambda = current entry,
 * row -= lambda * A_j (Alg 2, readings R8, R9).  Without
 * GBLA_FUSE_D the coefficients are stored as C' (mN x n_piv, the 4-step
 * variant P:689-698).  With GBLA_FUSE_D the B rows are applied in the same
 * pass (Alg 2) and D holds D - C A^-1 B on return. */
gbla_status gbla_reduce_C(gbla_mat h, uint32_t flags, void *stream);

/* Step 3 / 4-step variant step 4:
 * D <- D - C' B after an unfused gbla_reduce_C, or D <- D - C B' after
 * gbla_reduce_B.  Requires exactly one of them since gbla_splice
 * (GBLA_E_ORDER otherwise: both would give D - C A^-1 A^-1 B). */
gbla_status gbla_update_D(gbla_mat h, void *stream);

/* Step 4, fully reduced (reading R13): R = RREF(D) over GF(p):
 * rows sorted by pivot column, leading 1, zero in every other pivot column,
 * zero rows dropped.  *rank = rows(R); rank(M) = n_piv + rank.
 * Echelons the CURRENT D (callable after any of the above).  flags select
 * the trailing-update engine (GBLA_DENSE_TC default, GBLA_DENSE_INT).
 * GBLA_ECHELON_REF: skip the back elimination (rows are never reduced by
 * later pivots): R is then a row echelon form of D -- rows sorted by pivot
 * column, leading 1, zero below every pivot, the same pivot columns and rank
 * as the RREF, RREF(R) = the fully reduced result -- but not canonical (the
 * entries above later pivots depend on the panel boundaries).
 * Synchronizes `stream`. */
gbla_status gbla_echelon_D(gbla_mat h, uint32_t flags, void *stream, int64_t *rank);

/* the fully reduced row echelon form of the WHOLE M, in M's original
 * column order: after gbla_echelon_D (fully reduced), the pivot rows are
 * reduced to [I | B''] with B' = A^-1 B (Step 2) and B'' = B' - B'[:, pivcol] R
 * (the second reduction by the rows of R), and Step 5 puts the columns back in
 * the original order.  The result is RREF(M): rank(M) = n_piv + rank rows,
 * each with a leading 1, zero in every other pivot column, rows sorted by pivot column.
 * B' is computed on the tensor cores by the sparse phase itself (targets e_k give
 * -e_k A^-1 B); B'' by K11.  Stored in the handle as a device CSR (u64 row_ptr, u32
 * original columns ascending per row, u16 values); *rank_M = rows.  GBLA_E_ORDER before
 * gbla_echelon_D or after a GBLA_ECHELON_REF echelon; GBLA_E_INVAL on a row-sharded D.
 * Synchronizes `stream`.  Memory: n_piv x nN u16 (dense -B') plus the CSR. */
gbla_status gbla_rref_M(gbla_mat h, void *stream, int64_t *rank_M);
/* Device CSR view of RREF(M) (m = rank(M) rows, n = M's columns), valid until gbla_mat_free. */
gbla_status gbla_get_rref_M(gbla_mat h, gbla_csr *out);

/* The whole pipeline: splice -> (new order: fused reduce_C | standard:
 * reduce_B + update_D) -> echelon_D.  Returns the handle holding every
 * result.  Synchronizes `stream`. */
gbla_status gbla_reduce(gbla_ctx ctx, const gbla_csr *M, uint32_t p, uint32_t flags,
                        void *stream, gbla_mat *out);

/* K11 as a standalone op (used by the echelon; exposed for tests/benches):
 *   C[r_i, x] <- (C[r_i, x] - sum_{k<K} A[i, k] * B[k, x]) mod p,
 *   i < rows, x < cols, r_i = rowidx ? rowidx[i] : i.
 * A: rows x K (row stride lda), B: K x cols (stride ldb), C: stride ldc; all
 * device u16 residues < p; K <= 512.  engine 0 = tcgen05 (u8 limbs; K <= 128:
 * one K-block, else the multi-K kernel of the echelon's deferred updates;
 * exact: every s32 limb sum <= 512 * 255^2 * 2 < 2^31), 1 = INT pipe.
 * Synchronizes. */
gbla_status gbla_modgemm(gbla_ctx ctx, uint32_t p, int64_t rows, int64_t cols, int64_t K,
                         const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb,
                         const uint32_t *rowidx, uint16_t *C, int64_t ldc, int engine, void *stream);
/* K11 microbenchmark (roofline of the trailing update): device-generated
 * pseudo-random operand tiles and C (rows x cols, K <= 512), one untimed launch, then
 * `reps` launches timed by CUDA events on `stream`; *ms_per_launch = mean device time.
 * Work per launch: rows * cols * ceil(K/128)*128 modMACs (4 u8 MACs each). */
gbla_status gbla_modgemm_bench(gbla_ctx ctx, uint32_t p, int64_t rows, int64_t cols, int64_t K, int reps,
                               void *stream, float *ms_per_launch);

/* ---- wider prime fields --------------------- */
/* M over GF(p) with residues below 2^31: as gbla_csr with u32 values (1 <= val < p). */
typedef struct {
    int64_t m, n, nnz;
    const uint64_t *row_ptr;
    const uint32_t *col;
    const uint32_t *val;
} gbla_csr32;
/* The whole reduction for a prime 2 < p < 2^31 (the paper's float representation covers p < 2^23,
 * its library 32-bit residues too): Step 1 with readings R1-R7, Alg 2 (new order, readings R8/R9)
 * with u64 accumulators (delayed reduction when n_piv (p-1)^2 < 2^63, else reduced at every add),
 * the canonical RREF of D_new (R13) by column-by-column Gauss-Jordan -- all on the INT pipe with
 * u32 storage (the tensor-core pipeline is u16 / two u8 limbs).  flags: GBLA_HOST_INPUT only.
 * Results through gbla_get_dims / gbla_get_maps / gbla_get_opcount and gbla_get_wide; the u16
 * calls reject a wide handle (GBLA_E_ORDER).  GBLA_E_DOMAIN if p is not a prime in (2, 2^31),
 * GBLA_E_INVAL for malformed input.  Synchronizes `stream`. */
gbla_status gbla_reduce_wide(gbla_ctx ctx, const gbla_csr32 *M, uint32_t p, uint32_t flags, void *stream,
                             gbla_mat *out);
/* Results of gbla_reduce_wide (device pointers owned by h, row stride *ld): rank(D_new), pivcol[rank],
 * R (rank x nN, u32), D_new (mN x nN, u32). */
gbla_status gbla_get_wide(gbla_mat h, int64_t *rank, const uint32_t **pivcol, const uint32_t **R,
                          const uint32_t **Dnew, int64_t *ld);

/* ---- the paper's binary matrix formats -------- */
/* Format 1 (Table `tab:bin_formats`): m, n, p (u32), nnz (u64), data (u16 x nnz),
 * cols (u32 x nnz), rows (u32 x m, row lengths).  Format 2: b (u32: type code
 * u | (v << 1) of the pdata elements in the low 3 bits, 8 * 2^v bits, unsigned/signed; format
 * version in the top 8 bits, 0 or 1), m, n (u32), p, nnz (u64), rows (u32 x m), polmap (u32 x m),
 * k (u64), colid (u64 x k: a run of s > 1 consecutive columns from f as the slot pair f, s; a
 * single column f as f | 2^31), pnb (u32), pnnz (u64), prow (u32 x pnb), pdata.  Little-endian.
 * Readings R20, R23-R26 of DESIGN.md: the paper's "f AND (1 << 31)" is read as OR; its type code
 * example "011" for unsigned 16-bit is accepted beside 010. */
typedef struct {
    int32_t format;         /* 1 or 2 */
    uint32_t typecode;      /* Format 2: b & 7 */
    uint32_t version;       /* Format 2: b >> 24 */
    uint32_t p;
    int64_t m, n, nnz;
    int64_t k, pnb, pnnz;   /* Format 2 section sizes */
} gbla_file_info;
/* Parse and check the header of a file image (host bytes, len = the whole file): sizes of every
 * section must add up to len.  GBLA_E_INVAL on a malformed header, GBLA_E_DOMAIN for p >= 2^16. */
gbla_status gbla_file_info_parse(const void *bytes, size_t len, int format, gbla_file_info *out);
/* Decode a file image (host bytes) on the device into the caller's device CSR arrays:
 * row_ptr (m + 1), col (nnz), val (nnz) -- sizes from gbla_file_info_parse -- ready for
 * gbla_splice / gbla_reduce.  Format 2: column runs decoded by prefix sums over the colid slots
 * and every row's values expanded from its polynomial (polmap, prow, pdata) on the GPU.
 * GBLA_E_INVAL on content errors (counts, a run without its length, a polynomial length that
 * is not the row's, values outside [1, p)).  Synchronizes `stream`. */
gbla_status gbla_file_decode(gbla_ctx ctx, const void *bytes, size_t len, int format, uint64_t *row_ptr,
                             uint32_t *col, uint16_t *val, void *stream);

/* ---- results (views valid until gbla_mat_free) ------------------------- */
gbla_status gbla_get_dims(gbla_mat h, int64_t *npiv, int64_t *mN, int64_t *nN);
/* sigma[n]: column c -> sigma index; pivot_row[npiv]; nonpivot_row[mN]
 * (original row ids).  Device pointers. */
gbla_status gbla_get_maps(gbla_mat h, const uint32_t **sigma, const uint32_t **pivot_row,
                          const uint32_t **nonpivot_row);
/* Current dense D (mN x nN, row stride *ld elements), device. */
gbla_status gbla_get_D(gbla_mat h, const uint16_t **D, int64_t *ld);
/* C' (mN x npiv, stride *ld) after unfused reduce_C; NULL otherwise. */
gbla_status gbla_get_Cprime(gbla_mat h, const uint16_t **X, int64_t *ld);
/* B' (npiv x nN, stride *ld) after reduce_B; NULL otherwise. */
gbla_status gbla_get_Bprime(gbla_mat h, const uint16_t **Bp, int64_t *ld);
/* Densify an original quadrant ('A','B','C','D', normalized, sigma order)
 * into caller-provided device memory `out` (rows x cols, stride ld). */
gbla_status gbla_densify_quadrant(gbla_mat h, char which, uint16_t *out, int64_t ld, void *stream);
/* Two-row multilines of A|B (Definition, example P:524-556):
 * pair k = sigma-ordered pivot rows (2k, 2k+1) (the last pair of an odd
 * n_piv has a zero second row); its slots are q in [ptr[k], ptr[k+1]): col[q]
 * = a sigma column of the union of both supports (ascending, no column where
 * both rows are zero), val[q] = row 2k value (low 16 bits) | row 2k+1 value
 * (high 16 bits), explicit zeros allowed (the paper's `val`, interleaved per
 * column; `pos` = col).  Built on first call (enqueued on `stream`, which is
 * synchronized).  Device pointers, owned by h; *npairs = ceil(n_piv / 2). */
gbla_status gbla_get_multilines(gbla_mat h, void *stream, int64_t *npairs, const uint64_t **ptr,
                                const uint32_t **col, const uint32_t **val);
/* Column runs of the multilines (north star "device sparse-row format with column runs"; the
 * device analogue of Format 2's run compression (f, s)), built with them on first use:
 * the slots of pair k are cut into maximal runs of consecutive columns (also cut where the pair's
 * own diagonal-block columns end and where its N columns begin), runs [run_ptr[k], run_ptr[k+1]);
 * run r covers columns run_col[r] .. run_col[r] + run_len[r] - 1 at the pair's slots
 * run_slot[r] .. (relative to the pair's first slot; values in the multiline val array).  The
 * INT-pipe engine (GBLA_SPARSE_INT) walks these runs.  Device pointers owned by h. */
gbla_status gbla_get_multiline_runs(gbla_mat h, void *stream, int64_t *nruns, const uint64_t **run_ptr,
                                    const uint32_t **run_col, const uint32_t **run_len, const uint32_t **run_slot);
/* R (rank x nN, stride *ld) and pivcol[rank] after gbla_echelon_D. */
gbla_status gbla_get_rref(gbla_mat h, int64_t *rank, const uint32_t **pivcol,
                          const uint16_t **R, int64_t *ld);
/* Copy R (row-major, rank x nN, no padding) and pivcol to HOST memory. */
gbla_status gbla_copy_rref_to_host(gbla_mat h, uint32_t *pivcol, uint16_t *R, void *stream);
/* modMAC counts: sparse phase (Alg 2 count: for every nonzero lambda_j,
 * nnz(row_j) - 1) and the echelon's dense modMACs (algorithmic). */
gbla_status gbla_get_opcount(gbla_mat h, uint64_t *sparse_modmac, uint64_t *dense_modmac);
/* Per-phase device times in ms of the last calls on this handle
 * (splice, reduce_C, reduce_B, update_D, echelon). */
gbla_status gbla_get_phase_ms(gbla_mat h, float *ms5);
gbla_status gbla_sync(gbla_mat h);
void gbla_mat_free(gbla_mat h);
const char *gbla_last_error(void);
/* Device time of one kernel family, summed over its launches on this handle
 * (CUDA events on the handle's stream; recorded only when the environment
 * variable GBLA_KERNEL_TIMERS is set when the handle is created).  which:
 * 0 = K5' sweep (C' = C A^-1 block forward substitution, tcgen05),
 * 1 = K7' update (D -= C' B, tcgen05), 2 = K10 panel factorization,
 * 3 = K11 trailing update of the echelon (tcgen05), 4 = K11 new pivot rows,
 * 5 = K14 back substitution of the row echelon form (RREF = U_sq^-1 U by the
 * K5' sweep on the pivot block of U; its setup kernels included).
 * Synchronizes the handle's stream. */
gbla_status gbla_get_kernel_ms(gbla_mat h, int which, float *ms, int64_t *launches);
/* Algorithmic modMACs of the same kernel family on this handle (this rank):
 * 0 = Alg 2 A-part count (sum over nonzero lambda_j of nnz(A_j) - 1),
 * 1 = Alg 2 B-part count, 2 = sum over panels of candidates * kp * 128,
 * 3 = sum over panels of nrows * kp * width, 4 = sum of kp * kp * width,
 * 5 = back substitution: sum over the non-pivot columns q of R of r_q (r_q + 1) / 2,
 * r_q = pivots left of q (the modMACs of the triangular solve U_sq X = U_rest);
 * 6 = not modMACs: sum over panels of nrows * width, the D entries the
 * trailing updates read and write (the HBM roofline of K11). */
gbla_status gbla_get_kernel_work(gbla_mat h, int which, uint64_t *modmac);
/* u8 MACs the tensor cores executed for kernel family `which` (as in gbla_get_kernel_ms) on this
 * handle: 0 (K5' sweep) and 5 (K14 back substitution) count 4 x 128^3 per 128 x 128 tile pair of
 * the dense band tiles (limb products), whatever the tiles' density; the other families 0 (not
 * counted).  Executed / (4 x algorithmic) is the dense-tile overhead of the family. */
gbla_status gbla_get_kernel_exec(gbla_mat h, int which, uint64_t *u8macs);
/* Number of libgbla kernels launched by this process so far (diagnostics). */
uint64_t gbla_kernel_launches(void);
/* Library build/version string. */
const char *gbla_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GBLA_H */
