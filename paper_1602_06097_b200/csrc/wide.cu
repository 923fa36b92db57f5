// wide.cu -- SURVEY 8(f) f4: the reduction over wider prime fields, 2 < p < 2^31 (the paper's
// float representation covers p < 2^23 and its library also handles 32-bit residues).
//
// The u16 pipeline's kernels carry two u8 limbs per residue on the tensor cores and u16 storage;
// residues below 2^31 take this separate INT-pipe path with u32 storage and u64 arithmetic:
//   W1 k_w_scan     validate, lead, weight, inverse of the leading value (Fermat), pivot choice by
//                   atomicMin of (weight << 32 | row) (reading R1)
//   W2 k_w_cols / k_w_sigma / k_w_rows   pivot columns -> scan -> sigma (R2-R4); pivot and
//                   non-pivot rows (R5, R7)
//   W3 k_w_fill     sigma-ordered monic rows (R6), P entries first, CSR
//   W4 k_w_reduce   Alg 2 (R8/R9): a CTA per target, its dense u64 accumulator in global
//                   memory; lambda = acc[j] mod p captured, acc -= lambda * row_j; products are
//                   < 2^62, the accumulator is reduced at every add unless (p-1)^2 * n_piv < 2^63
//                   (then only when lambda is read and at output: delayed reduction); D_new in u32
//   W5 k_w_find / k_w_factor / k_w_elim / k_w_norm   canonical RREF of D_new (R13) by column-by-
//                   column Gauss-Jordan: for each column the first unused row with a nonzero entry
//                   becomes the pivot row, every other row eliminates the column, the pivot row is
//                   scaled to a leading 1; four launches per column, no host synchronization
//   W6 k_w_compact  R = the pivot rows in pivot-column order
// Barrett reduction (fmod64 of internal.cuh, m64 = floor(2^64 / p)) is exact for every p < 2^32.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t wmul(uint32_t a, uint32_t b, const Field &F)
{
    return fmod64((uint64_t)a * b, F);
}

// W1: one warp per row
__global__ void k_w_scan(int64_t m, int64_t n, int64_t nnz, const uint64_t *__restrict__ rp,
                         const uint32_t *__restrict__ col, const uint32_t *__restrict__ val, Field F,
                         uint32_t *__restrict__ lead, uint32_t *__restrict__ inv_lead,
                         unsigned long long *__restrict__ key, uint32_t *__restrict__ err)
{
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= m) return;
    const uint64_t s = rp[r], e = rp[r + 1];
    uint32_t bad = 0;
    if (e < s || e > (uint64_t)nnz) {
        bad = 1;
    } else {
        for (uint64_t q = s + lane; q < e; q += 32) {
            const uint32_t c = col[q], v = val[q];
            if ((int64_t)c >= n || (q > s && col[q - 1] >= c)) bad |= 2;
            if (v == 0 || v >= F.p) bad |= 4;
        }
    }
    bad = __reduce_or_sync(FULL, bad);
    if (lane) return;
    if (bad) {
        atomicOr(err, bad);
        lead[r] = GBLA_NONE;
    } else if (s == e) {
        lead[r] = GBLA_NONE;
    } else {
        lead[r] = col[s];
        inv_lead[r] = finv(val[s], F);
        atomicMin(&key[col[s]], ((unsigned long long)(e - s) << 32) | (unsigned long long)r);
    }
}

__global__ void k_w_cols(int64_t n, const unsigned long long *__restrict__ key, uint32_t *__restrict__ flag)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < n) flag[c] = key[c] != ~0ull;
    else if (c == n) flag[c] = 0;
}

__global__ void k_w_sigma(int64_t n, const unsigned long long *__restrict__ key, const uint32_t *__restrict__ pidx,
                          uint32_t *__restrict__ sigma, uint32_t *__restrict__ pivot_row, uint32_t *__restrict__ ispiv)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    const uint32_t npiv = pidx[n], k = pidx[c];
    if (key[c] != ~0ull) {
        sigma[c] = k;
        const uint32_t r = (uint32_t)(key[c] & 0xffffffffull);
        pivot_row[k] = r;
        ispiv[r] = 1;
    } else {
        sigma[c] = npiv + (uint32_t)(c - k);
    }
}

__global__ void k_w_rows(int64_t m, const uint32_t *__restrict__ ispiv, uint32_t *__restrict__ flag)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) flag[r] = ispiv[r] ? 0 : 1;
    else if (r == m) flag[r] = 0;
}

__global__ void k_w_nonpiv(int64_t m, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ idx,
                           uint32_t *__restrict__ nonpivot_row)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m && flag[r]) nonpivot_row[idx[r]] = (uint32_t)r;
}

__global__ void k_w_len(int64_t cnt, const uint32_t *__restrict__ rows, const uint64_t *__restrict__ rp,
                        uint64_t *__restrict__ len)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) len[i] = rp[rows[i] + 1] - rp[rows[i]];
    else if (i == cnt) len[i] = 0;
}

// W3: row i of the list -> sigma columns, monic values, the P entries (sigma < npiv) first in order
// (each group keeps its ascending order: sigma is monotone on P and on N); one warp per row
__global__ void k_w_fill(int64_t cnt, int64_t npiv, const uint32_t *__restrict__ rows, const uint64_t *__restrict__ rp,
                         const uint32_t *__restrict__ col, const uint32_t *__restrict__ val,
                         const uint32_t *__restrict__ inv_lead, const uint32_t *__restrict__ sigma, Field F,
                         const uint64_t *__restrict__ optr, uint32_t *__restrict__ ocol, uint32_t *__restrict__ oval,
                         uint32_t *__restrict__ onp)
{
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= cnt) return;
    const uint32_t r = rows[i];
    const uint64_t s = rp[r], e = rp[r + 1];
    const uint32_t inv = s < e ? inv_lead[r] : 1;
    uint32_t np = 0;
    for (uint64_t q = s + lane; q < e; q += 32) np += sigma[col[q]] < npiv;
    np = __reduce_add_sync(FULL, np);
    uint64_t oP = optr[i], oN = optr[i] + np;
    for (uint64_t base = s; base < e; base += 32) {
        const uint64_t q = base + lane;
        const bool live = q < e;
        const uint32_t sc = live ? sigma[col[q]] : 0;
        const bool isP = live && sc < npiv;
        const unsigned mP = __ballot_sync(FULL, isP), mN = __ballot_sync(FULL, live && !isP);
        const unsigned below = (1u << lane) - 1;
        if (live) {
            const uint64_t o = isP ? oP + __popc(mP & below) : oN + __popc(mN & below);
            ocol[o] = sc;
            oval[o] = wmul(val[q], inv, F);
        }
        oP += __popc(mP);
        oN += __popc(mN);
    }
    if (lane == 0) onp[i] = np;
}

// W4: Alg 2, a CTA per target (grid-stride), dense u64 accumulator acc[n] per CTA
__global__ void __launch_bounds__(256) k_w_reduce(int64_t mN, int64_t n, int64_t npiv, Field F, bool lazy,
                                                  const uint64_t *__restrict__ ab_ptr, const uint32_t *__restrict__ ab_col,
                                                  const uint32_t *__restrict__ ab_val, const uint64_t *__restrict__ cd_ptr,
                                                  const uint32_t *__restrict__ cd_col, const uint32_t *__restrict__ cd_val,
                                                  uint64_t *__restrict__ scratch, uint32_t *__restrict__ Dw, int64_t ldw,
                                                  unsigned long long *__restrict__ ops)
{
    uint64_t *acc = scratch + (size_t)blockIdx.x * n;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int64_t nN = n - npiv;
    unsigned long long myops = 0;
    for (int64_t t = blockIdx.x; t < mN; t += gridDim.x) {
        for (int64_t c = tid; c < n; c += nth) acc[c] = 0;
        __syncthreads();
        const uint64_t s = cd_ptr[t], e = cd_ptr[t + 1];
        for (uint64_t q = s + tid; q < e; q += nth) acc[cd_col[q]] = cd_val[q];
        __syncthreads();
        const int64_t j0 = s < e ? (int64_t)cd_col[s] : npiv;      // sigma(lead): the first (P) entry
        for (int64_t j = j0; j < npiv; j++) {
            const uint32_t lam = fmod64(acc[j], F);                 // captured before use (R9)
            __syncthreads();                                         // every thread has read acc[j]
            if (lam) {
                const uint64_t nl = F.p - lam;                       // subtract lambda * row_j (R8)
                const uint64_t a0 = ab_ptr[j], a1 = ab_ptr[j + 1];
                for (uint64_t q = a0 + tid; q < a1; q += nth) {
                    const uint64_t x = nl * ab_val[q];
                    uint64_t *y = acc + ab_col[q];
                    *y = lazy ? *y + x : fmod64(*y + x, F);
                }
                if (tid == 0) myops += a1 - a0 - 1;
            }
            __syncthreads();
        }
        for (int64_t c = tid; c < nN; c += nth) Dw[(size_t)t * ldw + c] = fmod64(acc[npiv + c], F);
        __syncthreads();
    }
    if (tid == 0 && myops) atomicAdd(ops, myops);
}

// W5: column-by-column Gauss-Jordan on Dw (mN x nN).  st[0] = pivot row of the current column
// (NONE if none), st[1] = its inverse, st[2] = rank so far.
__global__ void k_w_find(int64_t mN, int64_t c, Field F, const uint32_t *__restrict__ Dw, int64_t ldw,
                         uint32_t *__restrict__ used, uint32_t *__restrict__ st, uint32_t *__restrict__ pivrow,
                         uint32_t *__restrict__ pivcol)
{
    __shared__ uint32_t best;
    if (threadIdx.x == 0) best = GBLA_NONE;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < mN; i += blockDim.x)
        if (!used[i] && Dw[(size_t)i * ldw + c] != 0) atomicMin(&best, (uint32_t)i);
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t r = best;
        st[0] = r;
        if (r != GBLA_NONE) {
            st[1] = finv(Dw[(size_t)r * ldw + c], F);
            used[r] = 1;
            pivrow[st[2]] = r;
            pivcol[st[2]] = (uint32_t)c;
            st[2] += 1;
        }
    }
}

__global__ void k_w_factor(int64_t mN, int64_t c, const uint32_t *__restrict__ Dw, int64_t ldw,
                           const uint32_t *__restrict__ st, uint32_t *__restrict__ f)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (st[0] == GBLA_NONE || i >= mN) return;
    f[i] = (uint32_t)i == st[0] ? 0u : Dw[(size_t)i * ldw + c];
}

// D[i][x] -= f_i * inv * D[r][x] for x >= c (the pivot row itself unchanged here)
__global__ void k_w_elim(int64_t mN, int64_t nN, int64_t c, Field F, uint32_t *__restrict__ Dw, int64_t ldw,
                         const uint32_t *__restrict__ st, const uint32_t *__restrict__ f)
{
    const uint32_t r = st[0];
    if (r == GBLA_NONE) return;
    const int64_t i = blockIdx.y;
    for (int64_t i2 = i; i2 < mN; i2 += gridDim.y) {
        const uint32_t fi = f[i2];
        if (!fi) continue;
        const uint32_t g = wmul(fi, st[1], F);
        const uint32_t *pr = Dw + (size_t)r * ldw;
        uint32_t *row = Dw + (size_t)i2 * ldw;
        for (int64_t x = c + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nN; x += (int64_t)gridDim.x * blockDim.x) {
            const uint32_t s = wmul(g, pr[x], F);
            const uint32_t d = row[x];
            row[x] = d >= s ? d - s : d + F.p - s;
        }
    }
}

__global__ void k_w_norm(int64_t nN, int64_t c, Field F, uint32_t *__restrict__ Dw, int64_t ldw,
                         const uint32_t *__restrict__ st)
{
    const uint32_t r = st[0];
    if (r == GBLA_NONE) return;
    uint32_t *row = Dw + (size_t)r * ldw;
    for (int64_t x = c + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nN; x += (int64_t)gridDim.x * blockDim.x)
        row[x] = wmul(row[x], st[1], F);
}

__global__ void k_w_compact(int64_t rank, int64_t nN, const uint32_t *__restrict__ Dw, int64_t ldw,
                            const uint32_t *__restrict__ pivrow, uint32_t *__restrict__ Rw)
{
    const int64_t k = blockIdx.y;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nN; x += (int64_t)gridDim.x * blockDim.x)
        Rw[(size_t)k * ldw + x] = Dw[(size_t)pivrow[k] * ldw + x];
}

template <class T>
gbla_status wscan(gbla_mat h, const T *in, T *out, int64_t n)
{
    size_t tb = 0;
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, h->stream));
    void *t;
    GBLA_TRY(dalloc(h, tb + 16, &t));
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t, tb, in, out, (int)n, h->stream));
    return GBLA_OK;
}

static bool is_prime32(uint32_t p)
{
    if (p < 2) return false;
    for (uint32_t d = 2; (uint64_t)d * d <= p; d++)
        if (p % d == 0) return false;
    return true;
}

gbla_status wide_impl(gbla_mat h, const gbla_csr32 *M)
{
    cudaStream_t st = h->stream;
    const int64_t m = h->m, n = h->n, nnz = h->nnz;
    const Field F = h->F;
    unsigned long long *key;
    uint32_t *err, *cflag, *pidx, *rflag, *ridx, *ispiv, *lead, *inv_lead;
    GBLA_TRY(dalloc_t(h, m + 1, &lead));
    GBLA_TRY(dalloc_t(h, m + 1, &inv_lead));
    GBLA_TRY(dalloc_t(h, n + 1, &key));
    GBLA_TRY(dalloc_t(h, 4, &err));
    GBLA_TRY(dalloc_t(h, n + 1, &cflag));
    GBLA_TRY(dalloc_t(h, n + 1, &pidx));
    GBLA_TRY(dalloc_t(h, m + 1, &rflag));
    GBLA_TRY(dalloc_t(h, m + 1, &ridx));
    GBLA_TRY(dalloc_t(h, m + 1, &ispiv));
    GBLA_TRY(dalloc_t(h, n + 1, &h->sigma));
    GBLA_TRY(dalloc_t(h, n + 1, &h->pivot_row));
    GBLA_TRY(dalloc_t(h, m + 1, &h->nonpivot_row));
    GBLA_CUDA_TRY(cudaMemsetAsync(key, 0xff, (n + 1) * 8, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(err, 0, 16, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(ispiv, 0, (m + 1) * 4, st));
    if (m) k_w_scan<<<grid_for(m * 32, 256), 256, 0, st>>>(m, n, nnz, M->row_ptr, M->col, M->val, F, lead, inv_lead, key, err);
    k_w_cols<<<grid_for(n + 1, 256), 256, 0, st>>>(n, key, cflag);
    note_launch(2);
    GBLA_TRY(wscan<uint32_t>(h, cflag, pidx, n + 1));
    if (n) k_w_sigma<<<grid_for(n, 256), 256, 0, st>>>(n, key, pidx, h->sigma, h->pivot_row, ispiv);
    k_w_rows<<<grid_for(m + 1, 256), 256, 0, st>>>(m, ispiv, rflag);
    note_launch(2);
    GBLA_TRY(wscan<uint32_t>(h, rflag, ridx, m + 1));
    if (m) k_w_nonpiv<<<grid_for(m, 256), 256, 0, st>>>(m, rflag, ridx, h->nonpivot_row);
    note_launch();
    uint32_t hv[3];
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hv[0], err, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hv[1], pidx + n, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hv[2], ridx + m, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    if (hv[0]) {
        set_error("gbla_reduce_wide: invalid CSR input (code %u: 1=row_ptr, 2=column order/range, 4=value range)", hv[0]);
        return GBLA_E_INVAL;
    }
    const int64_t npiv = hv[1], mN = hv[2], nN = n - npiv;
    h->npiv = npiv;
    h->mN = mN;
    h->nN = nN;
    // W3: sigma-ordered monic rows of A|B (pivot order) and C|D (original order)
    uint64_t *len, *ab_ptr, *cd_ptr;
    uint32_t *ab_col, *ab_val, *cd_col, *cd_val, *np;
    GBLA_TRY(dalloc_t(h, (npiv > mN ? npiv : mN) + 1, &len));
    GBLA_TRY(dalloc_t(h, npiv + 1, &ab_ptr));
    GBLA_TRY(dalloc_t(h, mN + 1, &cd_ptr));
    GBLA_TRY(dalloc_t(h, (npiv > mN ? npiv : mN) + 1, &np));
    k_w_len<<<grid_for(npiv + 1, 256), 256, 0, st>>>(npiv, h->pivot_row, M->row_ptr, len);
    note_launch();
    GBLA_TRY(wscan<uint64_t>(h, len, ab_ptr, npiv + 1));
    k_w_len<<<grid_for(mN + 1, 256), 256, 0, st>>>(mN, h->nonpivot_row, M->row_ptr, len);
    note_launch();
    GBLA_TRY(wscan<uint64_t>(h, len, cd_ptr, mN + 1));
    uint64_t t64[2];
    GBLA_CUDA_TRY(cudaMemcpyAsync(&t64[0], ab_ptr + npiv, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&t64[1], cd_ptr + mN, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    GBLA_TRY(dalloc_t(h, t64[0] + 1, &ab_col));
    GBLA_TRY(dalloc_t(h, t64[0] + 1, &ab_val));
    GBLA_TRY(dalloc_t(h, t64[1] + 1, &cd_col));
    GBLA_TRY(dalloc_t(h, t64[1] + 1, &cd_val));
    if (npiv)
        k_w_fill<<<grid_for(npiv * 32, 256), 256, 0, st>>>(npiv, npiv, h->pivot_row, M->row_ptr, M->col, M->val,
                                                            inv_lead, h->sigma, F, ab_ptr, ab_col, ab_val, np);
    if (mN)
        k_w_fill<<<grid_for(mN * 32, 256), 256, 0, st>>>(mN, npiv, h->nonpivot_row, M->row_ptr, M->col, M->val,
                                                          inv_lead, h->sigma, F, cd_ptr, cd_col, cd_val, np);
    note_launch(2);
    // W4: D_new
    h->ldw = nN > 0 ? nN : 1;
    GBLA_TRY(dalloc_t(h, (size_t)(mN > 0 ? mN : 1) * h->ldw, &h->Dw));
    unsigned long long *ops;
    GBLA_TRY(dalloc_t(h, 1, &ops));
    GBLA_CUDA_TRY(cudaMemsetAsync(ops, 0, 8, st));
    if (mN && n) {
        int64_t grid = 4 * (int64_t)h->ctx->sm_count;
        if (grid > mN) grid = mN;
        uint64_t *scratch;
        GBLA_TRY(dalloc_t(h, (size_t)grid * n, &scratch));
        // delayed reduction when n_piv products of (p-1)^2 (plus a residue) stay below 2^63
        const bool lazy = (long double)(F.p - 1) * (long double)(F.p - 1) * (long double)(npiv + 1) < 9.2e18L;
        k_w_reduce<<<(unsigned)grid, 256, 0, st>>>(mN, n, npiv, F, lazy, ab_ptr, ab_col, ab_val, cd_ptr, cd_col, cd_val,
                                                   scratch, h->Dw, h->ldw, ops);
        note_launch();
    }
    // W5: RREF of D_new, on a copy (h->Dw keeps D_new)
    uint32_t *used, *stt, *pivrow, *f, *Dg;
    GBLA_TRY(dalloc_t(h, (size_t)(mN > 0 ? mN : 1) * h->ldw, &Dg));
    GBLA_CUDA_TRY(cudaMemcpyAsync(Dg, h->Dw, (size_t)(mN > 0 ? mN : 1) * h->ldw * 4, cudaMemcpyDeviceToDevice, st));
    GBLA_TRY(dalloc_t(h, mN + 1, &used));
    GBLA_TRY(dalloc_t(h, 4, &stt));
    GBLA_TRY(dalloc_t(h, mN + 1, &pivrow));
    GBLA_TRY(dalloc_t(h, mN + 1, &f));
    GBLA_TRY(dalloc_t(h, (mN < nN ? mN : nN) + 1, &h->pivcol));
    GBLA_CUDA_TRY(cudaMemsetAsync(used, 0, (mN + 1) * 4, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(stt, 0, 16, st));
    if (mN && nN) {
        for (int64_t c = 0; c < nN; c++) {
            k_w_find<<<1, 1024, 0, st>>>(mN, c, F, Dg, h->ldw, used, stt, pivrow, h->pivcol);
            k_w_factor<<<grid_for(mN, 256), 256, 0, st>>>(mN, c, Dg, h->ldw, stt, f);
            const unsigned gx = grid_for(nN - c, 256) < 8 ? grid_for(nN - c, 256) : 8;
            const unsigned gy = mN < 4096 ? (unsigned)mN : 4096u;
            k_w_elim<<<dim3(gx, gy), 256, 0, st>>>(mN, nN, c, F, Dg, h->ldw, stt, f);
            k_w_norm<<<gx, 256, 0, st>>>(nN, c, F, Dg, h->ldw, stt);
            note_launch(4);
        }
        GBLA_CUDA_TRY(cudaGetLastError());
    }
    uint32_t rk = 0;
    unsigned long long ov = 0;
    GBLA_CUDA_TRY(cudaMemcpyAsync(&rk, stt + 2, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&ov, ops, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->rank = rk;
    h->sparse_ops = ov;
    GBLA_TRY(dalloc_t(h, (size_t)(rk > 0 ? rk : 1) * h->ldw, &h->Rw));
    if (rk && nN) {
        for (int64_t k0 = 0; k0 < rk; k0 += 65535) {
            const int64_t cnt = rk - k0 < 65535 ? rk - k0 : 65535;
            k_w_compact<<<dim3(grid_for(nN, 256) < 8 ? grid_for(nN, 256) : 8, (unsigned)cnt), 256, 0, st>>>(
                cnt, nN, Dg, h->ldw, pivrow + k0, h->Rw + (size_t)k0 * h->ldw);
            note_launch();
        }
    }
    GBLA_CUDA_TRY(cudaGetLastError());
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    return GBLA_OK;
}

}  // namespace

extern "C" gbla_status gbla_reduce_wide(gbla_ctx ctx, const gbla_csr32 *M, uint32_t p, uint32_t flags, void *stream,
                                        gbla_mat *out)
{
    if (!out) { set_error("gbla_reduce_wide: out is NULL"); return GBLA_E_INVAL; }
    *out = nullptr;
    if (!ctx || !M) { set_error("gbla_reduce_wide: NULL argument"); return GBLA_E_INVAL; }
    if (flags & ~(uint32_t)GBLA_HOST_INPUT) { set_error("gbla_reduce_wide: unsupported flags 0x%x", flags); return GBLA_E_INVAL; }
    if (p <= 2 || p >= (1u << 31) || !is_prime32(p)) {
        set_error("gbla_reduce_wide: p = %u is not a prime in (2, 2^31)", p);
        return GBLA_E_DOMAIN;
    }
    if (M->m < 0 || M->n < 0 || M->nnz < 0 || M->m >= (1ll << 31) || M->n >= (1ll << 31) || !M->row_ptr ||
        (M->nnz > 0 && (!M->col || !M->val))) {
        set_error("gbla_reduce_wide: bad dimensions or NULL CSR array");
        return GBLA_E_INVAL;
    }
    GBLA_CUDA_TRY(cudaSetDevice(ctx->device));
    gbla_mat h = new gbla_mat_s();
    h->ctx = ctx;
    h->stream = (cudaStream_t)stream;
    h->p = p;
    h->F = make_field(p);
    h->wide = true;
    h->m = M->m;
    h->n = M->n;
    h->nnz = M->nnz;
    gbla_status s = GBLA_OK;
    gbla_csr32 dm = *M;
    if (flags & GBLA_HOST_INPUT) {
        uint64_t *rp = nullptr;
        uint32_t *c = nullptr, *v = nullptr;
        s = dalloc_t(h, M->m + 1, &rp);
        if (s == GBLA_OK) s = dalloc_t(h, M->nnz + 1, &c);
        if (s == GBLA_OK) s = dalloc_t(h, M->nnz + 1, &v);
        if (s == GBLA_OK &&
            (cudaMemcpyAsync(rp, M->row_ptr, (M->m + 1) * 8, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
             (M->nnz && (cudaMemcpyAsync(c, M->col, M->nnz * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
                         cudaMemcpyAsync(v, M->val, M->nnz * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)))) {
            set_error("gbla_reduce_wide: host copy failed");
            s = GBLA_E_CUDA;
        }
        dm.row_ptr = rp;
        dm.col = c;
        dm.val = v;
    }
    if (s == GBLA_OK) s = wide_impl(h, &dm);
    if (s != GBLA_OK) {
        gbla_mat_free(h);
        return s;
    }
    *out = h;
    return GBLA_OK;
}

extern "C" gbla_status gbla_get_wide(gbla_mat h, int64_t *rank, const uint32_t **pivcol, const uint32_t **R,
                                     const uint32_t **Dnew, int64_t *ld)
{
    if (!h) { set_error("NULL gbla_mat"); return GBLA_E_INVAL; }
    if (!h->wide) { set_error("gbla_get_wide: not a gbla_reduce_wide handle"); return GBLA_E_ORDER; }
    if (rank) *rank = h->rank;
    if (pivcol) *pivcol = h->pivcol;
    if (R) *R = h->Rw;
    if (Dnew) *Dnew = h->Dw;
    if (ld) *ld = h->ldw;
    return GBLA_OK;
}
