// fullrref.cu -- SURVEY 8(f) f2: the fully reduced row echelon form of the WHOLE M in its original
// column order, after gbla_echelon_D has produced R = RREF(D_new).
//
// The paper's route: Step 2 B' = A^-1 B, the second reduction of the pivot rows by R,
// B'' = B' - B'[:, pivcol(R)] R, and Step 5, the columns back in the original order
// (P:424-427).  The pivot rows become [I | B''] and the rows of R [0 | R]; sorted by pivot column
// they are RREF(M) (every pivot row keeps zeros left of its lead in the original order: A^-1 only
// combines rows whose leads lie to the right, and B'[i, q] = 0 for every R pivot q left of lead i).
//
// B' on the tensor cores, by the sparse phase itself: the targets e_k (one 1 at pivot column k,
// no N part) reduced by the pivot rows give X_k = e_k A^-1 and D_new_k = 0 - e_k A^-1 B = -B'_k,
// so an internal splice of [A|B ; I] (sigma column space, rows [0, npiv) forced to be the pivot
// rows) and the fused sweep + update produce -B' with the same kernels and exactness as D_new.
// Then -B'' = -B' - (-B'[:, pivcol]) R is one K11 product (K = rank, chunks of 512 on CTA pairs),
// and a compaction kernel writes RREF(M) as a CSR in the original column order.
#include <cub/cub.cuh>

#include "internal.cuh"

gbla_status reduce_c_tc(gbla_mat h, bool want_x16, bool fused);
void band_free(gbla_mat h);

namespace {

constexpr unsigned FULL = 0xffffffffu;

// row pointers of [A|B ; I] in sigma space: rows [0, npiv) are the sigma-ordered normalized pivot
// rows (h->ab_*), row npiv + k is e_k
__global__ void k_f2_rows(int64_t npiv, const uint64_t *__restrict__ ab_ptr, uint64_t nnz_ab,
                          uint64_t *__restrict__ rp, uint32_t *__restrict__ col, uint16_t *__restrict__ val)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > 2 * npiv) return;
    rp[i] = i <= npiv ? ab_ptr[i] : nnz_ab + (uint64_t)(i - npiv);
    if (i < npiv) {
        col[nnz_ab + i] = (uint32_t)i;
        val[nnz_ab + i] = 1;
    }
}

// A[k][r] = Bn[k][pivcol[r]] (the columns of -B' at R's pivots; a copy: the product updates Bn)
__global__ void k_gather_pcols(int64_t npiv, int64_t rank, const uint16_t *__restrict__ Bn, int64_t ldb,
                               const uint32_t *__restrict__ pivcol, uint16_t *__restrict__ A, int64_t lda)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rank) return;
    const uint32_t c = pivcol[r];
    for (int64_t k = blockIdx.y; k < npiv; k += gridDim.y) A[(size_t)k * lda + r] = Bn[(size_t)k * ldb + c];
}

// ncol[j] = original column of N column j (sigma index npiv + j)
__global__ void k_ncol(int64_t n, int64_t npiv, const uint32_t *__restrict__ sigma, uint32_t *__restrict__ ncol)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < n && sigma[c] >= npiv) ncol[sigma[c] - npiv] = (uint32_t)c;
}

__global__ void k_rpc(int64_t rank, const uint32_t *__restrict__ ncol, const uint32_t *__restrict__ pivcol,
                      uint32_t *__restrict__ rpc)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < rank) rpc[r] = ncol[pivcol[r]];
}

__device__ __forceinline__ int64_t lower_bound_u32(const uint32_t *a, int64_t n, uint32_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// output slot of every row (the two pivot-column lists are each ascending: merge by binary search)
// and its entry count; one warp per row.  Rows [0, npiv): pivot rows (1 at pcol[k], then the
// nonzeros of -(-B''_k)); rows npiv + r: R_r.
__global__ void k_rm_count(int64_t npiv, int64_t rank, int64_t nN, const uint32_t *__restrict__ pcol,
                           const uint32_t *__restrict__ rpc, const uint16_t *__restrict__ Bn, int64_t ldb,
                           const uint16_t *__restrict__ R, int64_t ldR, uint64_t *__restrict__ cnt,
                           uint32_t *__restrict__ slot)
{
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= npiv + rank) return;
    const bool prow = i < npiv;
    const uint16_t *row = prow ? Bn + (size_t)i * ldb : R + (size_t)(i - npiv) * ldR;
    uint32_t c = 0;
    for (int64_t x = lane; x < nN; x += 32) c += row[x] != 0;
    c = __reduce_add_sync(FULL, c);
    if (lane == 0) {
        const int64_t s = prow ? i + lower_bound_u32(rpc, rank, pcol[i])
                               : (i - npiv) + lower_bound_u32(pcol, npiv, rpc[i - npiv]);
        slot[i] = (uint32_t)s;
        cnt[s] = c + (prow ? 1 : 0);
    }
}

// fill: the row's entries in ascending original column (the pivot first), warp-compacted
__global__ void k_rm_fill(int64_t npiv, int64_t rank, int64_t nN, Field F, const uint32_t *__restrict__ pcol,
                          const uint32_t *__restrict__ ncol, const uint16_t *__restrict__ Bn, int64_t ldb,
                          const uint16_t *__restrict__ R, int64_t ldR, const uint32_t *__restrict__ slot,
                          const uint64_t *__restrict__ ptr, uint32_t *__restrict__ ocol, uint16_t *__restrict__ oval)
{
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= npiv + rank) return;
    const bool prow = i < npiv;
    const uint16_t *row = prow ? Bn + (size_t)i * ldb : R + (size_t)(i - npiv) * ldR;
    uint64_t o = ptr[slot[i]];
    if (prow) {
        if (lane == 0) {
            ocol[o] = pcol[i];
            oval[o] = 1;
        }
        o++;
    }
    for (int64_t x0 = 0; x0 < nN; x0 += 32) {
        const int64_t x = x0 + lane;
        uint32_t v = x < nN ? row[x] : 0;
        if (prow && v) v = F.p - v;                        // B'' = -(-B'')
        const unsigned m = __ballot_sync(FULL, v != 0);
        if (v) {
            const uint64_t q = o + __popc(m & ((1u << lane) - 1));
            ocol[q] = ncol[x];
            oval[q] = (uint16_t)v;
        }
        o += __popc(m);
    }
}

}  // namespace

// -B' = -(A^-1 B) on the tensor cores (see the header): a new internal handle whose D (npiv x nN,
// stride ldD) holds -B'.  The caller frees it with gbla_mat_free after the last kernel that reads it.
// The Alg 2 op count of the e_k targets is added to h->sparse_ops.
gbla_status neg_bprime_tc(gbla_mat h, const char *who, gbla_mat *out)
{
    cudaStream_t st = h->stream;
    const int64_t npiv = h->npiv, n = h->n;
    *out = nullptr;
    gbla_mat h2 = new gbla_mat_s();
    h2->ctx = h->ctx;
    h2->stream = st;
    h2->p = h->p;
    h2->F = h->F;
    h2->m = 2 * npiv;
    h2->n = n;
    h2->nnz = h->nnz_ab + npiv;
    h2->force_piv = npiv;
    uint64_t *rp = nullptr;
    uint32_t *col = nullptr;
    uint16_t *val = nullptr;
    gbla_status s = dalloc_t(h2, 2 * npiv + 1, &rp);
    if (s == GBLA_OK) s = dalloc_t(h2, (size_t)h2->nnz, &col);
    if (s == GBLA_OK) s = dalloc_t(h2, (size_t)h2->nnz, &val);
    if (s == GBLA_OK && h->nnz_ab) {
        if (cudaMemcpyAsync(col, h->ab_col, h->nnz_ab * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
            cudaMemcpyAsync(val, h->ab_val, h->nnz_ab * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
            set_error("%s: copy of the pivot rows failed", who);
            s = GBLA_E_CUDA;
        }
    }
    if (s == GBLA_OK) {
        k_f2_rows<<<grid_for(2 * npiv + 1, 256), 256, 0, st>>>(npiv, h->ab_ptr, (uint64_t)h->nnz_ab, rp, col, val);
        note_launch();
        const gbla_csr Mf{2 * npiv, n, h2->nnz, rp, col, val};
        s = splice_impl(h2, &Mf, 0);
    }
    if (s == GBLA_OK && (h2->npiv != npiv || h2->mN != npiv)) {
        set_error("%s: internal splice gave %lld pivots / %lld targets (expected %lld)", who,
                  (long long)h2->npiv, (long long)h2->mN, (long long)npiv);
        s = GBLA_E_INTERNAL;
    }
    if (s == GBLA_OK) s = reduce_c_tc(h2, false, true);      // h2->D = -B'
    if (s == GBLA_OK) h->sparse_ops += h2->sparse_ops;       // (the op count of this TRSM)
    if (s != GBLA_OK) {
        cudaStreamSynchronize(st);
        gbla_mat_free(h2);
        return s;
    }
    *out = h2;
    return GBLA_OK;
}

namespace {

// Bp[i][c] = -Bn[i][c] mod p
__global__ void k_negate_rows(int64_t rows, int64_t cols, Field F, const uint16_t *__restrict__ Bn, int64_t ldn,
                              uint16_t *__restrict__ Bp, int64_t ldp)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
        const uint32_t v = Bn[(size_t)i * ldn + c];
        Bp[(size_t)i * ldp + c] = (uint16_t)(v ? F.p - v : 0);
    }
}

}  // namespace

// Step 2 on the tensor cores: B' = A^-1 B = -(-B'), dense in h->Bp (the layout of
// reduce_b_int).  gbla_reduce_B's default; GBLA_TRSM_INT=1 keeps the INT-pipe K8.
gbla_status reduce_b_tc(gbla_mat h)
{
    cudaStream_t st = h->stream;
    h->ldB = (h->nN + 127) / 128 * 128;
    if (h->ldB == 0) h->ldB = 128;
    if (!h->Bp) GBLA_TRY(dalloc_t(h, (size_t)(h->npiv > 0 ? h->npiv : 1) * h->ldB, &h->Bp));
    GBLA_CUDA_TRY(cudaMemsetAsync(h->Bp, 0, (size_t)(h->npiv > 0 ? h->npiv : 1) * h->ldB * sizeof(uint16_t), st));
    if (h->npiv == 0 || h->nN == 0) return GBLA_OK;
    gbla_mat h2 = nullptr;
    GBLA_TRY(neg_bprime_tc(h, "gbla_reduce_B", &h2));
    dim3 g(grid_for(h->nN, 256), (unsigned)(h->npiv < 1184 ? h->npiv : 1184));
    k_negate_rows<<<g, 256, 0, st>>>(h->npiv, h->nN, h->F, h2->D, h2->ldD, h->Bp, h->ldB);
    note_launch();
    gbla_status s = GBLA_OK;
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("gbla_reduce_B: %s", cudaGetErrorString(cudaGetLastError()));
        s = GBLA_E_CUDA;
    }
    gbla_mat_free(h2);
    return s;
}

gbla_status full_rref_impl(gbla_mat h)
{
    cudaStream_t st = h->stream;
    const int64_t npiv = h->npiv, nN = h->nN, n = h->n, rank = h->rank;
    // ---- -B' on the tensor cores: internal splice of [A|B ; I] with forced pivot rows
    gbla_mat h2 = nullptr;
    uint16_t *Bn = nullptr;
    int64_t ldb = (nN + 127) / 128 * 128;
    if (ldb == 0) ldb = 128;
    gbla_status s = GBLA_OK;
    if (npiv > 0) {
        s = neg_bprime_tc(h, "gbla_rref_M", &h2);
        if (s == GBLA_OK) {
            Bn = h2->D;
            ldb = h2->ldD;
        }
        // ---- -B'' = -B' - (-B'[:, pivcol]) R  (K11, K = rank)
        if (s == GBLA_OK && rank > 0 && nN > 0) {
            uint16_t *A = nullptr;
            const int64_t lda = (rank + 7) / 8 * 8;
            s = dalloc_t(h2, (size_t)npiv * lda, &A);
            if (s == GBLA_OK) {
                dim3 g(grid_for(rank, 128), (unsigned)(npiv < 65535 ? npiv : 65535));
                k_gather_pcols<<<g, 128, 0, st>>>(npiv, rank, Bn, ldb, h->pivcol, A, lda);
                note_launch();
                s = modgemm_sub_chunked(h->ctx, st, h->F, npiv, nN, rank, A, lda, h->R, h->ldR, Bn, ldb);
            }
        }
    }
    // ---- RREF(M) as a CSR in the original column order, rows by pivot column (Step 5)
    const int64_t rows = npiv + rank;
    uint32_t *ncol = nullptr, *rpc = nullptr, *slot = nullptr;
    uint64_t *cnt = nullptr;
    if (s == GBLA_OK) s = dalloc_t(h, nN + 1, &ncol);
    if (s == GBLA_OK) s = dalloc_t(h, rank + 1, &rpc);
    if (s == GBLA_OK) s = dalloc_t(h, rows + 1, &slot);
    if (s == GBLA_OK) s = dalloc_t(h, rows + 1, &cnt);
    if (s == GBLA_OK) s = dalloc_t(h, rows + 1, &h->rm_ptr);
    if (s == GBLA_OK) {
        k_ncol<<<grid_for(n, 256), 256, 0, st>>>(n, npiv, h->sigma, ncol);
        if (rank > 0) k_rpc<<<grid_for(rank, 256), 256, 0, st>>>(rank, ncol, h->pivcol, rpc);
        note_launch(2);
        if (rows > 0) {
            k_rm_count<<<grid_for(rows * 32, 256), 256, 0, st>>>(npiv, rank, nN, h->pcol, rpc, Bn, ldb, h->R, h->ldR,
                                                                 cnt, slot);
            note_launch();
        }
        size_t tb = 0;
        if (cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, h->rm_ptr, (int)(rows + 1), st) != cudaSuccess) {
            set_error("gbla_rref_M: scan sizing failed");
            s = GBLA_E_CUDA;
        }
        void *tmp = nullptr;
        if (s == GBLA_OK) s = dalloc(h, tb + 16, &tmp);
        if (s == GBLA_OK && cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, h->rm_ptr, (int)(rows + 1), st) != cudaSuccess) {
            set_error("gbla_rref_M: scan failed");
            s = GBLA_E_CUDA;
        }
    }
    uint64_t total = 0;
    if (s == GBLA_OK && (cudaMemcpyAsync(&total, h->rm_ptr + rows, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                         cudaStreamSynchronize(st) != cudaSuccess)) {
        set_error("gbla_rref_M: %s", cudaGetErrorString(cudaGetLastError()));
        s = GBLA_E_CUDA;
    }
    if (s == GBLA_OK) s = dalloc_t(h, total + 1, &h->rm_col);
    if (s == GBLA_OK) s = dalloc_t(h, total + 1, &h->rm_val);
    if (s == GBLA_OK && rows > 0) {
        k_rm_fill<<<grid_for(rows * 32, 256), 256, 0, st>>>(npiv, rank, nN, h->F, h->pcol, ncol, Bn, ldb, h->R, h->ldR,
                                                            slot, h->rm_ptr, h->rm_col, h->rm_val);
        note_launch();
        if (cudaGetLastError() != cudaSuccess) { set_error("gbla_rref_M: launch failed"); s = GBLA_E_CUDA; }
    }
    if (s == GBLA_OK && cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("gbla_rref_M: %s", cudaGetErrorString(cudaGetLastError()));
        s = GBLA_E_CUDA;
    }
    if (h2) gbla_mat_free(h2);                                // (after every kernel that reads -B'')
    if (s == GBLA_OK) {
        h->rankM = rows;
        h->rm_nnz = (int64_t)total;
    }
    return s;
}
