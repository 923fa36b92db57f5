// internal.cuh -- shared internals of libgbla (CUDA path only; the oracle
// shares nothing with this file).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>
#include <string>
#include <vector>

#include "gbla.h"

#define GBLA_NONE 0xFFFFFFFFu

// ------------------------------------------------------------------ field
// GF(p), p < 2^16 prime.  Residues are kept in [0, p); products of two
// residues are < 2^32, so u64 accumulators hold >= 2^32 products before
// overflow (delayed reduction).  Reduction of a u64 uses Barrett
// with m64 = floor(2^64 / p): q = mulhi(x, m64) >= floor(x/p) - 1, so one
// conditional subtraction gives the canonical residue.
struct Field {
    uint32_t p;
    uint32_t c16;      // 2^16 mod p (< 2^15 for every p < 2^16: p > 2^15 gives 2^16 - p, else < p)
    uint64_t m64;
    uint32_t m32;      // floor((2^32 - 1) / p)
    uint32_t pad;
};

static inline Field make_field(uint32_t p) {
    Field F;
    F.p = p;
    F.c16 = (uint32_t)(65536u % p);
    F.m64 = ~0ull / p;
    F.m32 = 0xffffffffu / p;
    F.pad = 0;
    return F;
}

__device__ __forceinline__ uint32_t fmod64(uint64_t x, const Field &F) {
    uint64_t q = __umul64hi(x, F.m64);
    uint64_t r = x - q * (uint64_t)F.p;
    return (uint32_t)(r >= F.p ? r - F.p : r);
}
// v < 2^32 -> v mod p (32-bit Barrett: the quotient estimate is short by at most 1)
__device__ __forceinline__ uint32_t fmod32(uint32_t v, const Field &F) {
    const uint32_t r = v - __umulhi(v, F.m32) * F.p;
    return r >= F.p ? r - F.p : r;
}
// S = 2^16 hh + 2^8 xx + ll mod p from the three u8-limb accumulators of a tensor-core product
// (each < 2^31): with a, b = hh, xx mod p, t = a c16 + 256 b + ll < 2^30 + 2^24 + 2^31 < 2^32
// (a c16 <= p (2^16 - p) <= 2^30 for p > 2^15, < p^2 < 2^30 otherwise; ll needs no reduction),
// then t mod p.  32-bit arithmetic only.
__device__ __forceinline__ uint32_t fmod_limbs(uint32_t hh, uint32_t xx, uint32_t ll, const Field &F) {
    const uint32_t t = fmod32(hh, F) * F.c16 + (fmod32(xx, F) << 8) + ll;
    return fmod32(t, F);
}
// d - s mod p for two residues packed in 16-bit halves
__device__ __forceinline__ uint32_t fsub2(uint32_t d, uint32_t s, uint32_t p2) {
    return __vadd2(__vsub2(d, s), __vcmpltu2(d, s) & p2);
}
__device__ __forceinline__ uint32_t fmul(uint32_t a, uint32_t b, const Field &F) {
    return fmod64((uint64_t)a * b, F);
}
// a^(p-2) = a^-1 (Fermat; p prime).  a != 0.
__device__ __forceinline__ uint32_t finv(uint32_t a, const Field &F) {
    uint32_t e = F.p - 2, r = 1, b = a;
    while (e) {
        if (e & 1) r = fmul(r, b, F);
        b = fmul(b, b, F);
        e >>= 1;
    }
    return r;
}
__device__ __forceinline__ uint32_t fneg(uint32_t a, const Field &F) { return a ? F.p - a : 0; }

// ------------------------------------------------------------------ device errors
// Bounded spin-waits on inter-CTA flags (flags published by other CTAs of a persistent kernel, or
// by a kernel on another stream) must never hang the GPU nor continue silently: on a timeout they
// latch a code into the device error word of their translation unit and stop waiting; the host
// reads and clears the word when the phase ends and fails the call with GBLA_E_INTERNAL (the
// result is discarded).  GBLA_DEV_ERR_UNIT(fn) defines the word and the host check `fn`.
enum { DEVERR_GATHER_WAIT = 1, DEVERR_WIN_FLAG = 2, DEVERR_SWEEP_FLAG = 8 };
#define GBLA_DEV_ERR_UNIT(fn)                                                                      \
    static __device__ uint32_t g_dev_err = 0;                                                      \
    static __device__ __forceinline__ void dev_err_latch(uint32_t code) { atomicOr(&g_dev_err, code); } \
    gbla_status fn(cudaStream_t st, const char *where)                                             \
    {                                                                                              \
        uint32_t v = 0;                                                                            \
        if (cudaMemcpyFromSymbolAsync(&v, g_dev_err, 4, 0, cudaMemcpyDeviceToHost, st) != cudaSuccess || \
            cudaStreamSynchronize(st) != cudaSuccess) {                                            \
            set_error("%s: reading the device error word: %s", where, cudaGetErrorString(cudaGetLastError())); \
            return GBLA_E_CUDA;                                                                    \
        }                                                                                          \
        if (!v) return GBLA_OK;                                                                    \
        const uint32_t z = 0;                                                                      \
        cudaMemcpyToSymbolAsync(g_dev_err, &z, 4, 0, cudaMemcpyHostToDevice, st);                 \
        cudaStreamSynchronize(st);                                                                 \
        set_error("%s: an inter-CTA wait timed out on the device (code 0x%x); result discarded", where, v); \
        return GBLA_E_INTERNAL;                                                                    \
    }
gbla_status panel_dev_err(cudaStream_t st, const char *where);
gbla_status tcgemm_dev_err(cudaStream_t st, const char *where);
gbla_status sweep_dev_err(cudaStream_t st, const char *where);

// ------------------------------------------------------------------ launches
// Host-side count of libgbla kernel launches (bench.py reports it).
void note_launch(int n = 1);

// ------------------------------------------------------------------ errors
void set_error(const char *fmt, ...);
#define GBLA_CUDA_TRY(expr)                                                              \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
            return GBLA_E_CUDA;                                                          \
        }                                                                                \
    } while (0)
#define GBLA_TRY(expr)                      \
    do {                                    \
        gbla_status s_ = (expr);            \
        if (s_ != GBLA_OK) return s_;       \
    } while (0)

// ------------------------------------------------------------------ handles
struct gbla_ctx_s {
    int device = 0;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
    size_t smem_optin = 0;
    gbla_alloc_fn alloc = nullptr;
    gbla_free_fn free_fn = nullptr;
    void *user = nullptr;
    void *nccl_comm = nullptr;   // ncclComm_t
    int rank = 0, world = 1;
    // per-context resources reused across calls (creating them per call costs host time that
    // stalls the pipelined panel loop): the echelon's side stream, sync events, pinned scratch
    size_t (*memq)(void *) = nullptr;    // gbla_ctx_set_mem_query
    void *memq_user = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    void *pinned = nullptr;
    size_t pinned_bytes = 0;
};
cudaStream_t ctx_side_stream(gbla_ctx c);      // high priority, non-blocking; NULL on failure
cudaEvent_t ctx_event(gbla_ctx c, int i);      // i < 4, timing disabled
void *ctx_pinned(gbla_ctx c, size_t bytes);    // pinned host scratch (grows), NULL on failure

struct Alloc {
    void *ptr;
    size_t bytes;
};

// per-kernel-family CUDA-event timers (GBLA_KERNEL_TIMERS=1; gbla_get_kernel_ms)
enum { KT_SWEEP = 0, KT_UPDATE = 1, KT_PANEL = 2, KT_TRAIL = 3, KT_RN = 4, KT_BSUB = 5, KT_N = 6 };
struct KTimers {
    bool on = false;
    std::vector<cudaEvent_t> ev[KT_N];
};

struct gbla_mat_s {
    gbla_ctx ctx = nullptr;
    cudaStream_t stream = nullptr;
    int64_t m = 0, n = 0, nnz = 0, npiv = 0, mN = 0, nN = 0, npairs = 0;
    uint32_t p = 0;
    Field F{};

    // input (device); owned copy when the caller gave host memory
    const uint64_t *row_ptr = nullptr;
    const uint32_t *col = nullptr;
    const uint16_t *val = nullptr;

    // Step 1 maps
    uint32_t *lead = nullptr;          // [m]  first column or NONE
    uint16_t *inv_lead = nullptr;      // [m]  inverse of the leading value
    uint32_t *sigma = nullptr;         // [n]
    uint32_t *pivot_row = nullptr;     // [npiv]
    uint32_t *pcol = nullptr;          // [npiv] original column of pivot i
    uint32_t *nonpivot_row = nullptr;  // [mN]
    uint32_t *tlead = nullptr;         // [mN] sigma(lead) of each target (n for zero rows)
    uint32_t *order = nullptr;         // [mN] targets sorted by tlead (longest first)

    // sigma-ordered rows: A|B (pivot order) and C|D (original order)
    uint64_t *ab_ptr = nullptr; uint32_t *ab_col = nullptr; uint16_t *ab_val = nullptr;
    uint32_t *ab_np = nullptr;         // [npiv] entries with sigma col < npiv (A part)
    uint64_t *cd_ptr = nullptr; uint32_t *cd_col = nullptr; uint16_t *cd_val = nullptr;
    uint32_t *cd_np = nullptr;         // [mN]
    int64_t nnz_ab = 0, nnz_cd = 0;

    // two-row multilines of A|B: pair k = pivot rows (2k, 2k+1)
    uint64_t *ml_ptr = nullptr;        // [npairs+1] slot offsets
    uint32_t *ml_col = nullptr;        // [slots] union columns (sigma order)
    uint32_t *ml_val = nullptr;        // [slots] lo16 = row 2k value, hi16 = row 2k+1 value
    uint32_t *ml_np = nullptr;         // [npairs] slots with col < npiv
    uint32_t *ml_skip = nullptr;       // [npairs] leading slots with col <= 2k+1
    uint16_t *ml_a01 = nullptr;        // [npairs] A[2k][2k+1]
    uint32_t *ab_w = nullptr;          // [npiv] nnz of pivot row
    int64_t nslots = 0;
    // column runs of the multiline slots (splice.cu k_mlr_*): pair k has runs [mr_ptr[k], mr_ptr[k+1]);
    // run r = columns mr_col[r] .. + mr_len[r] - 1 at slots ml_ptr[k] + mr_rel[r] ..; the first run of
    // the N part / after the pair's own diagonal-block slots: mr_np[k] / mr_skip[k]
    uint64_t *mr_ptr = nullptr, *mr_skip = nullptr, *mr_np = nullptr;
    uint32_t *mr_col = nullptr, *mr_len = nullptr, *mr_rel = nullptr;
    int64_t nruns = 0;

    // dense matrices
    uint16_t *D = nullptr; int64_t ldD = 0;     // mN x nN (current D)
    uint16_t *X = nullptr; int64_t ldX = 0;     // C' (mN x npiv)
    uint16_t *Bp = nullptr; int64_t ldB = 0;    // B' (npiv x nN)
    uint16_t *R = nullptr; int64_t ldR = 0;     // rank x nN
    uint32_t *pivcol = nullptr;
    int64_t rank = -1;

    int64_t force_piv = 0;             // internal splices (f2): rows [0, force_piv) are the pivot rows
    // f4 (gbla_reduce_wide): residues below 2^31, u32 storage
    bool wide = false;
    uint32_t *Dw = nullptr, *Rw = nullptr;
    int64_t ldw = 0;

    // f2: RREF of the whole M, original column order (gbla_rref_M): device CSR, rows by pivot column
    int64_t rankM = -1, rm_nnz = 0;
    uint64_t *rm_ptr = nullptr;
    uint32_t *rm_col = nullptr;
    uint16_t *rm_val = nullptr;

    uint64_t *opcount = nullptr;       // [mN] per-target sparse modMACs
    uint64_t sparse_ops = 0, dense_ops = 0;
    uint64_t kwork[KT_N] = {0, 0, 0, 0, 0, 0};   // algorithmic modMACs per kernel family (this rank)
    uint64_t kexec[KT_N] = {0, 0, 0, 0, 0, 0};   // u8 MACs the tensor cores executed (dense tiles; 0 = not counted)
    uint64_t trail_elems = 0;                  // D entries the echelon's trailing updates read + write

    // call-order state
    bool did_reduce_B = false, did_cprime = false, did_update = false, did_fused = false;
    bool have_xt = false;              // C' held as tensor-core tiles (sparse_tc.cu)
    bool ref_only = false;             // GBLA_ECHELON_REF: no back elimination in the echelon
    bool dist_rows = false;            // D is row-sharded over the ranks (dist_sparse_phase)
    bool dist_phase = false;           // the sparse phase ran sharded (no band / C' for gbla_rref_M)
    float phase_ms[5] = {0, 0, 0, 0, 0};

    // tensor-core sparse path: dense band tiles of A|B, X tiles (sparse_tc.cu)
    struct BandTiles *bt = nullptr;

    KTimers kt;

    std::vector<Alloc> allocs;
};

// device memory through the context allocator, recorded on the handle
gbla_status dalloc(gbla_mat h, size_t bytes, void **out);
template <class T>
static inline gbla_status dalloc_t(gbla_mat h, size_t count, T **out) {
    return dalloc(h, count * sizeof(T) + 16, reinterpret_cast<void **>(out));
}
void dfree_all(gbla_mat h);
void dfree(gbla_mat h, void *p);      // release one allocation early
void *ctx_alloc(gbla_ctx c, size_t bytes, cudaStream_t s);
void ctx_free(gbla_ctx c, void *p, cudaStream_t s);

// phases
gbla_status splice_impl(gbla_mat h, const gbla_csr *M, uint32_t flags);
gbla_status reduce_c_int(gbla_mat h, bool fused, bool keep_x);
gbla_status update_d_from_x_int(gbla_mat h);
gbla_status reduce_b_int(gbla_mat h);
gbla_status reduce_b_tc(gbla_mat h);      // fullrref.cu: B' by the tensor-core sparse phase
gbla_status update_d_from_bp_int(gbla_mat h);
gbla_status echelon_impl(gbla_mat h, uint32_t flags);
gbla_status reduce_c_tc(gbla_mat h, bool want_x16, bool fused);
gbla_status update_d_tc(gbla_mat h);
void band_free(gbla_mat h);
void band_release(gbla_mat h);
gbla_status ensure_x(gbla_mat h);
gbla_status ensure_multilines(gbla_mat h);
// process-wide pool of timing events (creating events per mark costs host time
// that the panel loop cannot spare); events go back to the pool at gbla_mat_free
cudaEvent_t kt_event_get();
void kt_event_put(cudaEvent_t e);
static inline void kt_mark_on(gbla_mat h, int which, cudaStream_t s)
{
    if (!h->kt.on) return;
    if (s != h->stream && getenv("GBLA_KT_MAIN_ONLY")) return;
    cudaEvent_t e = kt_event_get();
    if (!e) return;
    cudaEventRecord(e, s);
    h->kt.ev[which].push_back(e);
}
static inline void kt_mark(gbla_mat h, int which) { kt_mark_on(h, which, h->stream); }
// one event closing a pair of family a and opening a pair of family b (adjacent launches: a second
// record between them would cut the programmatic-dependent-launch overlap)
static inline void kt_mark2(gbla_mat h, int a, int b, cudaStream_t s)
{
    if (!h->kt.on) return;
    if (s != h->stream && getenv("GBLA_KT_MAIN_ONLY")) return;
    cudaEvent_t e = kt_event_get();
    if (!e) return;
    cudaEventRecord(e, s);
    h->kt.ev[a].push_back(e);
    h->kt.ev[b].push_back(e);
}
// multi-GPU (dist.cu)
gbla_status dist_bcast_input(gbla_mat h, const gbla_csr *M, bool host_input, gbla_csr *out, gbla_status root_ok);
gbla_status dist_sparse_phase(gbla_mat h);
gbla_status dist_gather_dnew(gbla_mat h);   // replicated echelon: all of D_new on every rank
bool dist_echelon_replicated();             // GBLA_DIST_ECHELON != "panels"
gbla_status dist_check_async(gbla_ctx ctx);      // ncclCommGetAsyncError (aborts the comm on error)
int dist_emulated_world();
gbla_status densify_impl(gbla_mat h, char which, uint16_t *out, int64_t ld);
gbla_status full_rref_impl(gbla_mat h);
gbla_status modgemm_sub_chunked(gbla_ctx ctx, cudaStream_t st, const Field &F, int64_t rows, int64_t cols, int64_t K,
                                const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb, uint16_t *C, int64_t ldc);

// K11 launchers (tc_gemm.cu); see the kernels there for the argument conventions
gbla_status modgemm_tc_sub(cudaStream_t st, int64_t max_rows, const uint32_t *nrows_dev, int64_t cols, Field F,
                           const uint8_t *Alo, const uint8_t *Ahi, const uint8_t *Blo, const uint8_t *Bhi,
                           const uint32_t *rowidx, uint16_t *C, int64_t ldc, const int64_t *c0_dev,
                           const int64_t *win_dev, int64_t win_w, int ctsel, int grid_cap,
                           const int64_t *cend_dev = nullptr);
gbla_status modgemm_tc_sub_mk(cudaStream_t st, int64_t max_rows, const uint32_t *nrows_dev, int64_t cols, Field F,
                              const uint8_t *Alo, const uint8_t *Ahi, int64_t a_rt_stride, int nkb,
                              const uint8_t *Blo, const uint8_t *Bhi, int64_t b_kb_stride, const int64_t *kb_c0,
                              const uint32_t *rowidx, uint16_t *C, int64_t ldc, const int64_t *c0_dev,
                              const int64_t *win_dev, int64_t win_w, int ctsel, int grid_cap,
                              const uint8_t *B2lo = nullptr, const uint8_t *B2hi = nullptr);
gbla_status modgemm_tc_store(cudaStream_t st, int64_t cols, Field F, const uint8_t *Alo, const uint8_t *Ahi,
                             const uint8_t *Blo, const uint8_t *Bhi, uint16_t *O, int64_t ldo, uint8_t *Tlo,
                             uint8_t *Thi, const int64_t *c0_dev, const uint32_t *skip_dev, const int64_t *win_dev,
                             int64_t win_w, int ctsel, const uint32_t *orows = nullptr, int grid_cap = 0,
                             uint8_t *Tlo2 = nullptr, uint8_t *Thi2 = nullptr);
void modgemm_set_sms(int sms);
gbla_status modgemm_tc_win(cudaStream_t st, int64_t cols, Field F, const uint8_t *Tlo, const uint8_t *Thi,
                           const uint8_t *Bglo, const uint8_t *Bghi, uint8_t *Rlo, uint8_t *Rhi,
                           const uint8_t *Flo, const uint8_t *Fhi, const uint32_t *rows, const uint32_t *sel,
                           const uint32_t *nrows_dev, const uint32_t *kp_dev, const int64_t *c0_dev,
                           const int64_t *win_dev, int64_t win_w, uint16_t *D, int64_t ldD, uint32_t *flags,
                           uint32_t epoch, int grid, uint8_t *Rlo2 = nullptr, uint8_t *Rhi2 = nullptr);


// one-time per-device setup (function attributes): a bit per device ordinal, so a second context on
// another GPU of the same process sets them again
static inline unsigned long long dev_bit()
{
    int d = 0;
    cudaGetDevice(&d);
    return 1ull << (d & 63);
}

static inline unsigned grid_for(int64_t work, int per_block) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > 0x7fffffff) g = 0x7fffffff;
    return (unsigned)g;
}
