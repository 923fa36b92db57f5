#include <algorithm>
// api.cu -- the C ABI of include/gbla.h: argument checks, call-order state
// machine, allocation through the context allocator, phase timing.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

#include <atomic>
#include <mutex>

static thread_local char g_err[1024];
static std::atomic<unsigned long long> g_launches{0};

void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

// timing events, pooled per device (an event belongs to the device that was current when it was created)
static std::mutex g_ev_mu;
static std::vector<std::pair<int, cudaEvent_t>> g_ev_pool;

cudaEvent_t kt_event_get()
{
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_ev_mu);
        for (size_t i = g_ev_pool.size(); i-- > 0;)
            if (g_ev_pool[i].first == dev) {
                cudaEvent_t e = g_ev_pool[i].second;
                g_ev_pool.erase(g_ev_pool.begin() + i);
                return e;
            }
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    return e;
}

void kt_event_put(cudaEvent_t e)
{
    int dev = 0;
    cudaGetDevice(&dev);                  // callers return events on the device they were taken on
    std::lock_guard<std::mutex> lk(g_ev_mu);
    g_ev_pool.push_back({dev, e});
}

extern "C" uint64_t gbla_kernel_launches(void) { return g_launches.load(); }

void set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

extern "C" const char *gbla_last_error(void) { return g_err; }

extern "C" const char *gbla_version(void)
{
    return "libgbla 0.1 (sm_100a; Faugere-Lachartre over GF(p), p < 2^16; arXiv 1602.06097)";
}

void *ctx_alloc(gbla_ctx c, size_t bytes, cudaStream_t s)
{
    if (bytes == 0) bytes = 16;
    if (c->alloc) return c->alloc(bytes, (void *)s, c->user);
    void *p = nullptr;
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) return nullptr;
    return p;
}

void ctx_free(gbla_ctx c, void *p, cudaStream_t s)
{
    if (!p) return;
    if (c->free_fn) c->free_fn(p, (void *)s, c->user);
    else cudaFreeAsync(p, s);
}

gbla_status dalloc(gbla_mat h, size_t bytes, void **out)
{
    void *p = ctx_alloc(h->ctx, bytes, h->stream);
    if (!p) {
        cudaGetLastError();
        set_error("device allocation of %zu bytes failed", bytes);
        return GBLA_E_NOMEM;
    }
    h->allocs.push_back({p, bytes});
    *out = p;
    return GBLA_OK;
}

void dfree(gbla_mat h, void *p)
{
    if (!p) return;
    for (size_t i = 0; i < h->allocs.size(); i++)
        if (h->allocs[i].ptr == p) {
            ctx_free(h->ctx, p, h->stream);
            h->allocs.erase(h->allocs.begin() + i);
            return;
        }
}

void dfree_all(gbla_mat h)
{
    for (auto &a : h->allocs) ctx_free(h->ctx, a.ptr, h->stream);
    h->allocs.clear();
}

// ------------------------------------------------------------------ context
extern "C" gbla_status gbla_ctx_create(int device, gbla_ctx *out)
{
    if (!out) { set_error("gbla_ctx_create: out is NULL"); return GBLA_E_INVAL; }
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_error("gbla_ctx_create: no CUDA device (libgbla has no CPU fallback)");
        return GBLA_E_CUDA;
    }
    if (device < 0 || device >= ndev) { set_error("gbla_ctx_create: bad device %d", device); return GBLA_E_INVAL; }
    cudaDeviceProp prop;
    GBLA_CUDA_TRY(cudaSetDevice(device));
    GBLA_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error("gbla_ctx_create: device %d is sm_%d%d; libgbla is built for sm_100a only", device, prop.major,
                  prop.minor);
        return GBLA_E_CUDA;
    }
    gbla_ctx c = new gbla_ctx_s();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->cc_major = prop.major;
    c->cc_minor = prop.minor;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    *out = c;
    return GBLA_OK;
}

extern "C" gbla_status gbla_ctx_set_allocator(gbla_ctx ctx, gbla_alloc_fn alloc, gbla_free_fn free_fn, void *user)
{
    if (!ctx) { set_error("NULL context"); return GBLA_E_INVAL; }
    if ((alloc == nullptr) != (free_fn == nullptr)) { set_error("allocator needs both alloc and free"); return GBLA_E_INVAL; }
    ctx->alloc = alloc;
    ctx->free_fn = free_fn;
    ctx->user = user;
    return GBLA_OK;
}

extern "C" gbla_status gbla_ctx_set_mem_query(gbla_ctx ctx, gbla_memq_fn fn, void *user)
{
    if (!ctx) { set_error("NULL context"); return GBLA_E_INVAL; }
    ctx->memq = fn;
    ctx->memq_user = user;
    return GBLA_OK;
}

gbla_status dist_set_comm(gbla_ctx ctx, const void *id, int rank, int world);
void dist_destroy(gbla_ctx ctx);

extern "C" gbla_status gbla_ctx_set_comm(gbla_ctx ctx, const void *nccl_unique_id, int rank, int world)
{
    if (!ctx) { set_error("NULL context"); return GBLA_E_INVAL; }
    if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_unique_id)) {
        set_error("gbla_ctx_set_comm: bad rank %d / world %d", rank, world);
        return GBLA_E_INVAL;
    }
    return dist_set_comm(ctx, nccl_unique_id, rank, world);
}

cudaStream_t ctx_side_stream(gbla_ctx c)
{
    if (!c->side) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi) != cudaSuccess) {
            cudaGetLastError();
            c->side = nullptr;
        }
    }
    return c->side;
}

cudaEvent_t ctx_event(gbla_ctx c, int i)
{
    if (!c->ev[i] && cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        c->ev[i] = nullptr;
    }
    return c->ev[i];
}

void *ctx_pinned(gbla_ctx c, size_t bytes)
{
    if (c->pinned_bytes < bytes) {
        if (c->pinned) cudaFreeHost(c->pinned);
        c->pinned = nullptr;
        c->pinned_bytes = 0;
        if (cudaMallocHost(&c->pinned, bytes) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        c->pinned_bytes = bytes;
    }
    return c->pinned;
}

extern "C" void gbla_ctx_destroy(gbla_ctx ctx)
{
    if (!ctx) return;
    dist_destroy(ctx);
    cudaSetDevice(ctx->device);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    for (cudaEvent_t e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    delete ctx;
}

// ------------------------------------------------------------------ helpers
static bool is_prime_u32(uint32_t p)
{
    if (p < 2) return false;
    for (uint32_t d = 2; (uint64_t)d * d <= p; d++)
        if (p % d == 0) return false;
    return true;
}

// CUDA-event timer of one phase of the C ABI, also an NVTX range of the same name (host timeline;
// free when no tool is attached: nvtx3 is header-only and resolves its hooks lazily)
struct PhaseTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    explicit PhaseTimer(cudaStream_t st, const char *name = "gbla") : s(st) {
        nvtxRangePushA(name);
        a = kt_event_get();
        b = kt_event_get();
        if (a) cudaEventRecord(a, s);
    }
    float stop() {
        float ms = 0;
        if (!a || !b) return 0;
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    }
    ~PhaseTimer() {
        if (a) kt_event_put(a);
        if (b) kt_event_put(b);
        nvtxRangePop();
    }
};

static gbla_status check_mat(gbla_mat h, void *stream)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (h->wide) { set_error("a gbla_reduce_wide handle: use gbla_get_wide"); return GBLA_E_ORDER; }
    h->stream = (cudaStream_t)stream;
    GBLA_CUDA_TRY(cudaSetDevice(h->ctx->device));
    return GBLA_OK;
}

// ------------------------------------------------------------------ calls
extern "C" gbla_status gbla_splice(gbla_ctx ctx, const gbla_csr *M, uint32_t p, uint32_t flags, void *stream,
                                   gbla_mat *out)
{
    if (!out) { set_error("gbla_splice: out is NULL"); return GBLA_E_INVAL; }
    *out = nullptr;
    if (!ctx || !M) { set_error("gbla_splice: NULL argument"); return GBLA_E_INVAL; }
    if (flags & ~(uint32_t)GBLA_HOST_INPUT) { set_error("gbla_splice: unsupported flags 0x%x", flags); return GBLA_E_INVAL; }
    if (p <= 2 || p >= 65536 || !is_prime_u32(p)) {
        set_error("gbla_splice: p = %u is not a prime in (2, 2^16)", p);
        return GBLA_E_DOMAIN;
    }
    // with a communicator the splice is collective: rank 0's M is broadcast (C1)
    const bool dist = ctx->nccl_comm != nullptr;
    // rank 0's verdict on M travels with the dims broadcast, so every rank returns the same error
    // instead of the other ranks waiting forever in the collective
    gbla_status vs = GBLA_OK;
    if (!dist || ctx->rank == 0) {
        if (M->m < 0 || M->n < 0 || M->nnz < 0 || M->m >= (1ll << 31) || M->n >= (1ll << 31)) {
            set_error("gbla_splice: bad dimensions m=%lld n=%lld nnz=%lld", (long long)M->m, (long long)M->n,
                      (long long)M->nnz);
            vs = GBLA_E_INVAL;
        } else if (!M->row_ptr || (M->nnz > 0 && (!M->col || !M->val))) {
            set_error("gbla_splice: NULL CSR array");
            vs = GBLA_E_INVAL;
        }
        if (vs != GBLA_OK && !dist) return vs;
    }
    GBLA_CUDA_TRY(cudaSetDevice(ctx->device));
    gbla_mat h = new gbla_mat_s();
    h->ctx = ctx;
    h->stream = (cudaStream_t)stream;
    h->p = p;
    h->F = make_field(p);
    h->kt.on = getenv("GBLA_KERNEL_TIMERS") != nullptr;
    PhaseTimer tm(h->stream, "gbla_splice");
    gbla_status s;
    if (dist) {
        gbla_csr dm;
        s = dist_bcast_input(h, M, (flags & GBLA_HOST_INPUT) != 0, &dm, vs);
        if (s == GBLA_OK) {
            h->m = dm.m; h->n = dm.n; h->nnz = dm.nnz;
            s = splice_impl(h, &dm, 0);
        }
    } else {
        h->m = M->m; h->n = M->n; h->nnz = M->nnz;
        s = splice_impl(h, M, flags);
    }
    if (s != GBLA_OK) {
        cudaStreamSynchronize(h->stream);
        cudaGetLastError();
        dfree_all(h);
        band_free(h);
        delete h;
        return s;
    }
    h->phase_ms[0] = tm.stop();
    *out = h;
    return GBLA_OK;
}


extern "C" gbla_status gbla_reduce_C(gbla_mat h, uint32_t flags, void *stream)
{
    GBLA_TRY(check_mat(h, stream));
    if (flags & ~(uint32_t)(GBLA_FUSE_D | GBLA_KEEP_CPRIME | GBLA_SPARSE_INT)) {
        set_error("gbla_reduce_C: unsupported flags 0x%x", flags);
        return GBLA_E_INVAL;
    }
    if (h->did_cprime || h->did_fused) { set_error("gbla_reduce_C: already reduced"); return GBLA_E_ORDER; }
    const bool fused = flags & GBLA_FUSE_D;
    if (fused && (h->did_reduce_B || h->did_update)) {
        set_error("gbla_reduce_C(FUSE_D) after reduce_B/update_D would reduce D twice");
        return GBLA_E_ORDER;
    }
    PhaseTimer tm(h->stream, "gbla_reduce_C");
    const bool keep_x = (flags & GBLA_KEEP_CPRIME) != 0;
    if (flags & GBLA_SPARSE_INT) {
        GBLA_TRY(reduce_c_int(h, fused, keep_x));
    } else {
        // tensor-core block path (sparse_tc.cu): C' tiles, then D -= C' B
        GBLA_TRY(reduce_c_tc(h, keep_x || !fused, fused));
    }
    h->phase_ms[1] = tm.stop();
    if (fused) { h->did_fused = true; h->did_update = true; if (flags & GBLA_KEEP_CPRIME) h->did_cprime = true; }
    else h->did_cprime = true;
    return GBLA_OK;
}

extern "C" gbla_status gbla_reduce_B(gbla_mat h, void *stream)
{
    GBLA_TRY(check_mat(h, stream));
    if (h->did_reduce_B) { set_error("gbla_reduce_B: already done"); return GBLA_E_ORDER; }
    PhaseTimer tm(h->stream, "gbla_reduce_B");
    // default: the tensor-core sparse phase on the targets e_k (fullrref.cu); GBLA_TRSM_INT=1: K8
    const char *te = getenv("GBLA_TRSM_INT");
    const bool trsm_int = te && atoi(te) != 0;
    if (trsm_int) GBLA_TRY(reduce_b_int(h));
    else GBLA_TRY(reduce_b_tc(h));
    h->phase_ms[2] = tm.stop();
    h->did_reduce_B = true;
    return GBLA_OK;
}

extern "C" gbla_status gbla_update_D(gbla_mat h, void *stream)
{
    GBLA_TRY(check_mat(h, stream));
    if (h->did_update) { set_error("gbla_update_D: D already updated"); return GBLA_E_ORDER; }
    const bool have_x = h->did_cprime, have_b = h->did_reduce_B;
    if (have_x == have_b) {
        set_error(have_x ? "gbla_update_D: both reduce_B and reduce_C were run (would give D - C A^-1 A^-1 B)"
                         : "gbla_update_D: needs reduce_B or an unfused reduce_C first");
        return GBLA_E_ORDER;
    }
    PhaseTimer tm(h->stream, "gbla_update_D");
    if (have_x && h->have_xt) GBLA_TRY(update_d_tc(h));
    else if (have_x) GBLA_TRY(update_d_from_x_int(h));
    else GBLA_TRY(update_d_from_bp_int(h));
    h->phase_ms[3] = tm.stop();
    h->did_update = true;
    return GBLA_OK;
}

extern "C" gbla_status gbla_echelon_D(gbla_mat h, uint32_t flags, void *stream, int64_t *rank)
{
    GBLA_TRY(check_mat(h, stream));
    if (flags & ~(uint32_t)(GBLA_DENSE_INT | GBLA_DENSE_TC | GBLA_ECHELON_REF)) {
        set_error("gbla_echelon_D: unsupported flags 0x%x", flags);
        return GBLA_E_INVAL;
    }
    if (h->rank >= 0) { set_error("gbla_echelon_D: already echelonized"); return GBLA_E_ORDER; }
    PhaseTimer tm(h->stream, "gbla_echelon_D");
    GBLA_TRY(echelon_impl(h, flags));
    h->phase_ms[4] = tm.stop();
    if (rank) *rank = h->rank;
    return GBLA_OK;
}

extern "C" gbla_status gbla_rref_M(gbla_mat h, void *stream, int64_t *rank_M)
{
    GBLA_TRY(check_mat(h, stream));
    if (h->rank < 0) { set_error("gbla_rref_M: needs gbla_echelon_D first"); return GBLA_E_ORDER; }
    if (h->ref_only) { set_error("gbla_rref_M: needs the fully reduced R (not GBLA_ECHELON_REF)"); return GBLA_E_ORDER; }
    if (h->dist_rows || h->dist_phase) {
        set_error("gbla_rref_M: single-GPU only (the sparse phase ran sharded)");
        return GBLA_E_INVAL;
    }
    if (h->rankM < 0) GBLA_TRY(full_rref_impl(h));
    if (rank_M) *rank_M = h->rankM;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_rref_M(gbla_mat h, gbla_csr *out)
{
    if (!h || !out) { set_error("gbla_get_rref_M: NULL argument"); return GBLA_E_INVAL; }
    if (h->rankM < 0) { set_error("gbla_get_rref_M: call gbla_rref_M first"); return GBLA_E_ORDER; }
    out->m = h->rankM;
    out->n = h->n;
    out->nnz = h->rm_nnz;
    out->row_ptr = h->rm_ptr;
    out->col = h->rm_col;
    out->val = h->rm_val;
    return GBLA_OK;
}

extern "C" gbla_status gbla_reduce(gbla_ctx ctx, const gbla_csr *M, uint32_t p, uint32_t flags, void *stream,
                                   gbla_mat *out)
{
    if (!out) { set_error("gbla_reduce: out is NULL"); return GBLA_E_INVAL; }
    *out = nullptr;
    if (flags & ~(uint32_t)GBLA_FLAGS_ALL) { set_error("gbla_reduce: unsupported flags 0x%x", flags); return GBLA_E_INVAL; }
    gbla_mat h = nullptr;
    GBLA_TRY(gbla_splice(ctx, M, p, flags & GBLA_HOST_INPUT, stream, &h));
    gbla_status s;
    const bool dist = ctx->nccl_comm != nullptr || dist_emulated_world() > 1;
    // (the INT-pipe echelon is single-GPU only: with GBLA_DENSE_INT every rank reduces the whole D)
    if (dist && !(flags & (GBLA_ORDER_STANDARD | GBLA_SPARSE_INT | GBLA_KEEP_CPRIME | GBLA_DENSE_INT))) {
        // multi-GPU (dist.cu): row-sharded tensor-core sparse phase + D_new all-gather
        PhaseTimer tm(h->stream, "gbla_reduce:sharded_sparse_phase");
        s = dist_sparse_phase(h);
        h->did_fused = h->did_update = true;
        h->dist_rows = h->dist_phase = true;
        if (s == GBLA_OK && dist_echelon_replicated()) s = dist_gather_dnew(h);   // C7
        h->phase_ms[1] = tm.stop();
    } else if (flags & GBLA_ORDER_STANDARD) {
        s = gbla_reduce_B(h, stream);
        if (s == GBLA_OK) s = gbla_update_D(h, stream);
    } else {
        s = gbla_reduce_C(h, GBLA_FUSE_D | (flags & (GBLA_KEEP_CPRIME | GBLA_SPARSE_INT)), stream);
    }
    if (s == GBLA_OK)
        s = gbla_echelon_D(h, flags & (GBLA_DENSE_INT | GBLA_DENSE_TC | GBLA_ECHELON_REF), stream, nullptr);
    if (s != GBLA_OK) { gbla_mat_free(h); return s; }
    *out = h;
    return GBLA_OK;
}

// ------------------------------------------------------------------ results
extern "C" gbla_status gbla_get_dims(gbla_mat h, int64_t *npiv, int64_t *mN, int64_t *nN)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (npiv) *npiv = h->npiv;
    if (mN) *mN = h->mN;
    if (nN) *nN = h->nN;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_maps(gbla_mat h, const uint32_t **sigma, const uint32_t **pivot_row,
                                     const uint32_t **nonpivot_row)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (sigma) *sigma = h->sigma;
    if (pivot_row) *pivot_row = h->pivot_row;
    if (nonpivot_row) *nonpivot_row = h->nonpivot_row;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_D(gbla_mat h, const uint16_t **D, int64_t *ld)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (D) *D = h->D;
    if (ld) *ld = h->ldD;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_Cprime(gbla_mat h, const uint16_t **X, int64_t *ld)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (X) *X = h->did_cprime ? h->X : nullptr;
    if (ld) *ld = h->ldX;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_Bprime(gbla_mat h, const uint16_t **Bp, int64_t *ld)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (Bp) *Bp = h->did_reduce_B ? h->Bp : nullptr;
    if (ld) *ld = h->ldB;
    return GBLA_OK;
}

extern "C" gbla_status gbla_densify_quadrant(gbla_mat h, char which, uint16_t *out, int64_t ld, void *stream)
{
    GBLA_TRY(check_mat(h, stream));
    if (!out) { set_error("densify: out is NULL"); return GBLA_E_INVAL; }
    return densify_impl(h, which, out, ld);
}

extern "C" gbla_status gbla_get_multilines(gbla_mat h, void *stream, int64_t *npairs, const uint64_t **ptr,
                                           const uint32_t **col, const uint32_t **val)
{
    GBLA_TRY(check_mat(h, stream));
    GBLA_TRY(ensure_multilines(h));
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (npairs) *npairs = h->npairs;
    if (ptr) *ptr = h->ml_ptr;
    if (col) *col = h->ml_col;
    if (val) *val = h->ml_val;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_multiline_runs(gbla_mat h, void *stream, int64_t *nruns, const uint64_t **run_ptr,
                                               const uint32_t **run_col, const uint32_t **run_len,
                                               const uint32_t **run_slot)
{
    GBLA_TRY(check_mat(h, stream));
    GBLA_TRY(ensure_multilines(h));
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (nruns) *nruns = h->nruns;
    if (run_ptr) *run_ptr = h->mr_ptr;
    if (run_col) *run_col = h->mr_col;
    if (run_len) *run_len = h->mr_len;
    if (run_slot) *run_slot = h->mr_rel;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_rref(gbla_mat h, int64_t *rank, const uint32_t **pivcol, const uint16_t **R,
                                     int64_t *ld)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (h->rank < 0 || h->wide) { set_error("gbla_get_rref: echelon_D not run (or a wide handle)"); return GBLA_E_ORDER; }
    if (rank) *rank = h->rank;
    if (pivcol) *pivcol = h->pivcol;
    if (R) *R = h->R;
    if (ld) *ld = h->ldR;
    return GBLA_OK;
}

extern "C" gbla_status gbla_copy_rref_to_host(gbla_mat h, uint32_t *pivcol, uint16_t *R, void *stream)
{
    GBLA_TRY(check_mat(h, stream));
    if (h->rank < 0) { set_error("gbla_copy_rref_to_host: echelon_D not run"); return GBLA_E_ORDER; }
    if (h->rank == 0) return GBLA_OK;
    if (pivcol) GBLA_CUDA_TRY(cudaMemcpyAsync(pivcol, h->pivcol, h->rank * 4, cudaMemcpyDeviceToHost, h->stream));
    if (R && h->nN)
        GBLA_CUDA_TRY(cudaMemcpy2DAsync(R, h->nN * 2, h->R, h->ldR * 2, h->nN * 2, h->rank, cudaMemcpyDeviceToHost,
                                        h->stream));
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_opcount(gbla_mat h, uint64_t *sparse_modmac, uint64_t *dense_modmac)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (sparse_modmac) *sparse_modmac = h->sparse_ops;
    if (dense_modmac) *dense_modmac = h->dense_ops;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_phase_ms(gbla_mat h, float *ms5)
{
    if (!h || !ms5) { set_error("NULL argument"); return GBLA_E_INVAL; }
    memcpy(ms5, h->phase_ms, sizeof h->phase_ms);
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_kernel_ms(gbla_mat h, int which, float *ms, int64_t *launches)
{
    if (!h || which < 0 || which >= KT_N) { set_error("gbla_get_kernel_ms: bad argument"); return GBLA_E_INVAL; }
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    const auto &v = h->kt.ev[which];
    float tot = 0;
    for (size_t i = 0; i + 1 < v.size(); i += 2) {
        float t = 0;
        GBLA_CUDA_TRY(cudaEventElapsedTime(&t, v[i], v[i + 1]));
        tot += t;
    }
    if (ms) *ms = tot;
    if (launches) *launches = (int64_t)(v.size() / 2);
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_kernel_work(gbla_mat h, int which, uint64_t *modmac)
{
    if (!h || which < 0 || which > KT_N || !modmac) { set_error("gbla_get_kernel_work: bad argument"); return GBLA_E_INVAL; }
    *modmac = which == KT_N ? h->trail_elems : h->kwork[which];
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_kernel_exec(gbla_mat h, int which, uint64_t *u8macs)
{
    if (!h || which < 0 || which >= KT_N || !u8macs) { set_error("gbla_get_kernel_exec: bad argument"); return GBLA_E_INVAL; }
    *u8macs = h->kexec[which];
    return GBLA_OK;
}

extern "C" gbla_status gbla_sync(gbla_mat h)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    return GBLA_OK;
}

extern "C" void gbla_mat_free(gbla_mat h)
{
    if (!h) return;
    cudaSetDevice(h->ctx->device);
    // every kernel of this handle is done before its memory goes back to the allocator (the echelon
    // joins its side streams before returning, so h->stream covers them)
    cudaStreamSynchronize(h->stream);
    dfree_all(h);
    band_free(h);
    std::vector<cudaEvent_t> all;                 // an event shared by two timer pairs goes back once
    for (auto &v : h->kt.ev) all.insert(all.end(), v.begin(), v.end());
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    for (cudaEvent_t e : all) kt_event_put(e);
    delete h;
}
