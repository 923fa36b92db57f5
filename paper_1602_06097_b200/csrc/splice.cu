// splice.cu -- Step 1 of the Faugere-Lachartre reduction (P:359-378,
// P:219-229) on the device, and the device formats of the quadrants.
//
//   K1 k_scan_rows     validate rows, lead, weight, inverse of the leading
//                      value; atomicMin of (weight<<32 | row) into key[lead]
//                      picks the pivot row of each pivot column (reading R1)
//   K3 k_col_flags/k_sigma   pivot-column flags -> exclusive scan -> sigma
//   K4 k_fill_rows     normalized sigma-ordered rows of A|B and C|D
//      k_ml_count/k_ml_fill  two-row multilines of A|B
//      k_densify       dense D quadrant
#include <cub/cub.cuh>

#include "internal.cuh"

namespace {

constexpr unsigned FULL = 0xffffffffu;

// K1: one warp per row.
// nforce > 0 (internal splices only, f2): rows [0, nforce) win their pivot column whatever their
// weight (key weight 0); the public splice passes 0 (reading R1).
__global__ void k_scan_rows(int64_t m, int64_t n, int64_t nnz, const uint64_t *__restrict__ rp,
                            const uint32_t *__restrict__ col, const uint16_t *__restrict__ val, Field F,
                            uint32_t *__restrict__ lead, uint16_t *__restrict__ inv_lead,
                            unsigned long long *__restrict__ key, uint32_t *__restrict__ err, int64_t nforce)
{
    int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (r >= m) return;
    uint64_t s = rp[r], e = rp[r + 1];
    uint32_t bad = 0;
    if (e < s || e > (uint64_t)nnz) {
        bad = 1;
    } else {
        for (uint64_t q = s + lane; q < e; q += 32) {
            uint32_t c = col[q];
            uint32_t v = val[q];
            if ((int64_t)c >= n) bad |= 2;
            if (q > s && col[q - 1] >= c) bad |= 2;
            if (v == 0 || v >= F.p) bad |= 4;
        }
    }
    bad = __reduce_or_sync(FULL, bad);
    if (lane == 0) {
        if (bad) {
            atomicOr(err, bad);
            lead[r] = GBLA_NONE;
            inv_lead[r] = 0;
        } else if (s == e) {
            lead[r] = GBLA_NONE;   // zero row: goes to C|D (reading R7)
            inv_lead[r] = 0;
        } else {
            uint32_t c = col[s];
            lead[r] = c;
            inv_lead[r] = (uint16_t)finv(val[s], F);
            unsigned long long k = ((unsigned long long)(r < nforce ? 0 : e - s) << 32) | (unsigned long long)r;
            atomicMin(&key[c], k);
        }
    }
}

__global__ void k_col_flags(int64_t n, const unsigned long long *__restrict__ key, uint32_t *__restrict__ flag)
{
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < n) flag[c] = key[c] != ~0ull;
    else if (c == n) flag[c] = 0;
}

// sigma: P ascending -> 0..npiv-1, N ascending -> npiv.. (readings R3, R4)
__global__ void k_sigma(int64_t n, const unsigned long long *__restrict__ key, const uint32_t *__restrict__ pidx,
                        uint32_t *__restrict__ sigma, uint32_t *__restrict__ pivot_row, uint32_t *__restrict__ pcol)
{
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    uint32_t npiv = pidx[n];
    uint32_t k = pidx[c];
    if (key[c] != ~0ull) {
        sigma[c] = k;
        pivot_row[k] = (uint32_t)(key[c] & 0xffffffffull);
        pcol[k] = (uint32_t)c;
    } else {
        sigma[c] = npiv + (uint32_t)(c - k);
    }
}

__global__ void k_row_flags(int64_t m, const uint32_t *__restrict__ lead, const unsigned long long *__restrict__ key,
                            uint32_t *__restrict__ flag)
{
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) {
        uint32_t l = lead[r];
        bool is_piv = l != GBLA_NONE && (uint32_t)(key[l] & 0xffffffffull) == (uint32_t)r;
        flag[r] = !is_piv;
    } else if (r == m) {
        flag[r] = 0;
    }
}

__global__ void k_nonpivot(int64_t m, int64_t n, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ idx,
                           const uint32_t *__restrict__ lead, const uint32_t *__restrict__ sigma,
                           uint32_t *__restrict__ nonpivot_row, uint32_t *__restrict__ tlead)
{
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m || !flag[r]) return;
    uint32_t k = idx[r];
    nonpivot_row[k] = (uint32_t)r;
    uint32_t l = lead[r];
    tlead[k] = l == GBLA_NONE ? (uint32_t)n : sigma[l];
}

__global__ void k_row_len(int64_t nrows, const uint32_t *__restrict__ rows, const uint64_t *__restrict__ rp,
                          uint64_t *__restrict__ len)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nrows) {
        uint32_t r = rows[i];
        len[i] = rp[r + 1] - rp[r];
    } else if (i == nrows) {
        len[i] = 0;
    }
}

// K4: normalized rows in sigma order: P entries first, then N entries (both
// keep their relative order since sigma is increasing on P and on N).
// One warp per row.
__global__ void k_fill_rows(int64_t nrows, int64_t npiv, const uint32_t *__restrict__ rows,
                            const uint64_t *__restrict__ rp, const uint32_t *__restrict__ col,
                            const uint16_t *__restrict__ val, const uint16_t *__restrict__ inv_lead,
                            const uint32_t *__restrict__ sigma, Field F, const uint64_t *__restrict__ optr,
                            uint32_t *__restrict__ ocol, uint16_t *__restrict__ oval, uint32_t *__restrict__ onp)
{
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= nrows) return;
    uint32_t r = rows[i];
    uint64_t s = rp[r], e = rp[r + 1], o = optr[i];
    uint32_t il = inv_lead[r];
    unsigned lt = (1u << lane) - 1u;
    uint32_t base = 0;
    for (int pass = 0; pass < 2; pass++) {
        // four 32-slot chunks per step: their column and sigma loads are in flight together
        for (uint64_t q0 = s; q0 < e; q0 += 128) {
            uint32_t c[4], sc[4], v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint64_t q = q0 + 32 * u + lane;
                c[u] = q < e ? col[q] : 0xffffffffu;
                v[u] = q < e ? val[q] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) sc[u] = c[u] != 0xffffffffu ? sigma[c[u]] : 0xffffffffu;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const bool take = sc[u] != 0xffffffffu && ((sc[u] < (uint64_t)npiv) == (pass == 0));
                const unsigned msk = __ballot_sync(FULL, take);
                if (take) {
                    const uint32_t pos = base + __popc(msk & lt);
                    ocol[o + pos] = sc[u];
                    oval[o + pos] = (uint16_t)fmod32(v[u] * il, F);   // < 2^32: 32-bit Barrett
                }
                base += __popc(msk);
            }
        }
        if (pass == 0 && lane == 0) onp[i] = base;
    }
}

// Multiline pairs: union of the sigma-sorted supports of pivot
// rows 2k and 2k+1.  One thread per pair, sequential merge.
__global__ void k_ml_count(int64_t npairs, int64_t npiv, const uint64_t *__restrict__ ab_ptr,
                           const uint32_t *__restrict__ ab_col, uint64_t *__restrict__ cnt,
                           uint32_t *__restrict__ np, uint32_t *__restrict__ skip)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npairs) {
        if (k == npairs) cnt[k] = 0;
        return;
    }
    int64_t r0 = 2 * k, r1 = 2 * k + 1;
    uint64_t a = ab_ptr[r0], ae = ab_ptr[r0 + 1];
    uint64_t b = r1 < npiv ? ab_ptr[r1] : 0, be = r1 < npiv ? ab_ptr[r1 + 1] : 0;
    uint64_t c = 0;
    uint32_t nP = 0, nskip = 0;
    while (a < ae || b < be) {
        uint32_t ca = a < ae ? ab_col[a] : 0xffffffffu;
        uint32_t cb = b < be ? ab_col[b] : 0xffffffffu;
        uint32_t cc = ca < cb ? ca : cb;
        if (ca == cc) a++;
        if (cb == cc) b++;
        if (cc < (uint64_t)npiv) nP++;
        if (cc < (uint64_t)npiv && cc <= (uint64_t)r1) nskip++;   // the pair's own diagonal block
        c++;
    }
    cnt[k] = c;
    np[k] = nP;
    skip[k] = nskip;
}

__global__ void k_ml_fill(int64_t npairs, int64_t npiv, const uint64_t *__restrict__ ab_ptr,
                          const uint32_t *__restrict__ ab_col, const uint16_t *__restrict__ ab_val,
                          const uint64_t *__restrict__ ml_ptr, uint32_t *__restrict__ ml_col,
                          uint32_t *__restrict__ ml_val, uint16_t *__restrict__ a01)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npairs) return;
    int64_t r0 = 2 * k, r1 = 2 * k + 1;
    uint64_t a = ab_ptr[r0], ae = ab_ptr[r0 + 1];
    uint64_t b = r1 < npiv ? ab_ptr[r1] : 0, be = r1 < npiv ? ab_ptr[r1 + 1] : 0;
    uint64_t o = ml_ptr[k];
    uint16_t v01 = 0;
    while (a < ae || b < be) {
        uint32_t ca = a < ae ? ab_col[a] : 0xffffffffu;
        uint32_t cb = b < be ? ab_col[b] : 0xffffffffu;
        uint32_t cc = ca < cb ? ca : cb;
        uint32_t v0 = 0, v1 = 0;
        if (ca == cc) v0 = ab_val[a++];
        if (cb == cc) v1 = ab_val[b++];
        if (r1 < npiv && cc == (uint32_t)r1) v01 = (uint16_t)v0;
        ml_col[o] = cc;
        ml_val[o] = v0 | (v1 << 16);
        o++;
    }
    a01[k] = v01;
}

// Column runs of the multilines (north star "device sparse-row format with column runs"; the
// device analogue of Format 2's run compression (f, s)): the slots of pair k are cut into
// maximal runs of consecutive columns, also cut where the pair's own diagonal-block slots end
// (ml_skip) and where its N part begins (ml_np), so every consumer's slot range is a run range.
// Run r: start column mr_col[r], length mr_len[r], first slot ml_ptr[k] + mr_rel[r].  One warp per
// pair; runs found by ballots over the slots (count pass, then fill pass).
__device__ __forceinline__ bool ml_run_start(const uint32_t *col, uint64_t q, uint64_t q0, uint64_t qs, uint64_t qn)
{
    return q == q0 || q == qs || q == qn || col[q] != col[q - 1] + 1;
}
__global__ void k_mlr_count(int64_t npairs, const uint64_t *__restrict__ ml_ptr, const uint32_t *__restrict__ ml_col,
                            const uint32_t *__restrict__ ml_skip, const uint32_t *__restrict__ ml_np,
                            uint64_t *__restrict__ cnt)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k > npairs) return;
    if (k == npairs) { if (lane == 0) cnt[k] = 0; return; }
    const uint64_t q0 = ml_ptr[k], q1 = ml_ptr[k + 1], qs = q0 + ml_skip[k], qn = q0 + ml_np[k];
    uint32_t c = 0;
    for (uint64_t q = q0 + lane; q < q1; q += 32) c += ml_run_start(ml_col, q, q0, qs, qn);
    c = __reduce_add_sync(FULL, c);
    if (lane == 0) cnt[k] = c;
}
__global__ void k_mlr_fill(int64_t npairs, const uint64_t *__restrict__ ml_ptr, const uint32_t *__restrict__ ml_col,
                           const uint32_t *__restrict__ ml_skip, const uint32_t *__restrict__ ml_np,
                           const uint64_t *__restrict__ mr_ptr, uint32_t *__restrict__ mr_col,
                           uint32_t *__restrict__ mr_len, uint32_t *__restrict__ mr_rel,
                           uint64_t *__restrict__ mr_skip, uint64_t *__restrict__ mr_np)
{
    const int lane = threadIdx.x & 31;
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k >= npairs) return;
    const uint64_t q0 = ml_ptr[k], q1 = ml_ptr[k + 1], qs = q0 + ml_skip[k], qn = q0 + ml_np[k];
    uint64_t r = mr_ptr[k];                           // next run index of this pair
    if (lane == 0) { mr_skip[k] = mr_ptr[k + 1]; mr_np[k] = mr_ptr[k + 1]; }
    __syncwarp();
    for (uint64_t base = q0; base < q1; base += 32) {
        const uint64_t q = base + lane;
        const bool st = q < q1 && ml_run_start(ml_col, q, q0, qs, qn);
        const unsigned m = __ballot_sync(FULL, st);
        if (st) {
            const uint64_t ri = r + __popc(m & ((1u << lane) - 1));
            mr_col[ri] = ml_col[q];
            mr_rel[ri] = (uint32_t)(q - q0);
            if (q == qs) mr_skip[k] = ri;
            if (q == qn) mr_np[k] = ri;
        }
        r += __popc(m);
    }
    __syncwarp();
    // lengths: next run's first slot (or the pair's end) minus this run's
    for (uint64_t ri = mr_ptr[k] + lane; ri < mr_ptr[k + 1]; ri += 32) {
        const uint64_t e = ri + 1 < mr_ptr[k + 1] ? mr_rel[ri + 1] : q1 - q0;
        mr_len[ri] = (uint32_t)(e - mr_rel[ri]);
    }
    // a boundary at the pair's end (no skip / N slots) is the end index, set above
    if (lane == 0) {
        if (qs >= q1) mr_skip[k] = mr_ptr[k + 1];
        if (qn >= q1) mr_np[k] = mr_ptr[k + 1];
    }
}

// w[i] = nnz of sigma-ordered pivot row i
__global__ void k_row_w(int64_t npiv, const uint64_t *__restrict__ ab_ptr, uint32_t *__restrict__ w)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npiv) w[i] = (uint32_t)(ab_ptr[i + 1] - ab_ptr[i]);
}

// Densify part of the sigma-ordered rows: entries with sigma col in
// [c_lo, c_hi) go to out[i*ld + (col - c_lo)].  One warp per row.
__global__ void k_densify(int64_t nrows, const uint64_t *__restrict__ ptr, const uint32_t *__restrict__ colv,
                          const uint16_t *__restrict__ valv, int64_t c_lo, int64_t c_hi,
                          uint16_t *__restrict__ out, int64_t ld)
{
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= nrows) return;
    for (uint64_t q = ptr[i] + lane; q < ptr[i + 1]; q += 32) {
        int64_t c = colv[q];
        if (c >= c_lo && c < c_hi) out[i * ld + (c - c_lo)] = valv[q];
    }
}

__global__ void k_iota(int64_t n, uint32_t *__restrict__ a)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (uint32_t)i;
}

template <class T>
gbla_status exclusive_scan(gbla_mat h, const T *in, T *out, int64_t count)
{
    size_t tmp = 0;
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)count, h->stream));
    void *t = nullptr;
    GBLA_TRY(dalloc(h, tmp + 16, &t));
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)count, h->stream));
    return GBLA_OK;
}

}  // namespace

gbla_status densify_impl(gbla_mat h, char which, uint16_t *out, int64_t ld)
{
    cudaStream_t st = h->stream;
    int64_t rows, c_lo, c_hi;
    const uint64_t *ptr;
    const uint32_t *cv;
    const uint16_t *vv;
    switch (which) {
        case 'A': rows = h->npiv; c_lo = 0; c_hi = h->npiv; ptr = h->ab_ptr; cv = h->ab_col; vv = h->ab_val; break;
        case 'B': rows = h->npiv; c_lo = h->npiv; c_hi = h->n; ptr = h->ab_ptr; cv = h->ab_col; vv = h->ab_val; break;
        case 'C': rows = h->mN; c_lo = 0; c_hi = h->npiv; ptr = h->cd_ptr; cv = h->cd_col; vv = h->cd_val; break;
        case 'D': rows = h->mN; c_lo = h->npiv; c_hi = h->n; ptr = h->cd_ptr; cv = h->cd_col; vv = h->cd_val; break;
        default: set_error("densify: unknown quadrant '%c'", which); return GBLA_E_INVAL;
    }
    if (rows == 0 || c_hi == c_lo) return GBLA_OK;
    GBLA_CUDA_TRY(cudaMemset2DAsync(out, (size_t)ld * 2, 0, (size_t)(c_hi - c_lo) * 2, (size_t)rows, st));
    k_densify<<<grid_for(rows * 32, 256), 256, 0, st>>>(rows, ptr, cv, vv, c_lo, c_hi, out, ld); note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

gbla_status splice_impl(gbla_mat h, const gbla_csr *M, uint32_t flags)
{
    cudaStream_t st = h->stream;
    const int64_t m = h->m, n = h->n, nnz = h->nnz;

    // device copy of host input (e2e path)
    if (flags & GBLA_HOST_INPUT) {
        uint64_t *rp; uint32_t *c; uint16_t *v;
        GBLA_TRY(dalloc_t(h, m + 1, &rp));
        GBLA_TRY(dalloc_t(h, nnz, &c));
        GBLA_TRY(dalloc_t(h, nnz, &v));
        GBLA_CUDA_TRY(cudaMemcpyAsync(rp, M->row_ptr, (m + 1) * 8, cudaMemcpyHostToDevice, st));
        if (nnz) {
            GBLA_CUDA_TRY(cudaMemcpyAsync(c, M->col, nnz * 4, cudaMemcpyHostToDevice, st));
            GBLA_CUDA_TRY(cudaMemcpyAsync(v, M->val, nnz * 2, cudaMemcpyHostToDevice, st));
        }
        h->row_ptr = rp; h->col = c; h->val = v;
    } else {
        h->row_ptr = M->row_ptr; h->col = M->col; h->val = M->val;
    }

    unsigned long long *key;
    uint32_t *err, *cflag, *pidx, *rflag, *ridx;
    GBLA_TRY(dalloc_t(h, m + 1, &h->lead));
    GBLA_TRY(dalloc_t(h, m + 1, &h->inv_lead));
    GBLA_TRY(dalloc_t(h, n + 1, &key));
    GBLA_TRY(dalloc_t(h, 4, &err));
    GBLA_TRY(dalloc_t(h, n + 1, &cflag));
    GBLA_TRY(dalloc_t(h, n + 1, &pidx));
    GBLA_TRY(dalloc_t(h, m + 1, &rflag));
    GBLA_TRY(dalloc_t(h, m + 1, &ridx));
    GBLA_TRY(dalloc_t(h, n + 1, &h->sigma));
    GBLA_TRY(dalloc_t(h, n + 1, &h->pivot_row));
    GBLA_TRY(dalloc_t(h, n + 1, &h->pcol));
    GBLA_TRY(dalloc_t(h, m + 1, &h->nonpivot_row));
    GBLA_TRY(dalloc_t(h, m + 1, &h->tlead));
    GBLA_CUDA_TRY(cudaMemsetAsync(key, 0xff, (n + 1) * 8, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(err, 0, 16, st));

    if (m > 0)
        k_scan_rows<<<grid_for(m * 32, 256), 256, 0, st>>>(m, n, nnz, h->row_ptr, h->col, h->val, h->F, h->lead,
                                                          h->inv_lead, key, err, h->force_piv); note_launch();
    k_col_flags<<<grid_for(n + 1, 256), 256, 0, st>>>(n, key, cflag); note_launch();
    GBLA_TRY(exclusive_scan<uint32_t>(h, cflag, pidx, n + 1));
    k_sigma<<<grid_for(n, 256), 256, 0, st>>>(n, key, pidx, h->sigma, h->pivot_row, h->pcol); note_launch();
    k_row_flags<<<grid_for(m + 1, 256), 256, 0, st>>>(m, h->lead, key, rflag); note_launch();
    GBLA_TRY(exclusive_scan<uint32_t>(h, rflag, ridx, m + 1));
    k_nonpivot<<<grid_for(m, 256), 256, 0, st>>>(m, n, rflag, ridx, h->lead, h->sigma, h->nonpivot_row, h->tlead); note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());

    uint32_t hv[3];
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hv[0], err, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hv[1], pidx + n, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hv[2], ridx + m, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    if (hv[0]) {
        set_error("gbla_splice: invalid CSR input (code %u: 1=row_ptr, 2=column order/range, 4=value range)", hv[0]);
        return GBLA_E_INVAL;
    }
    h->npiv = hv[1];
    h->mN = hv[2];
    h->nN = n - h->npiv;
    h->npairs = (h->npiv + 1) / 2;
    const int64_t npiv = h->npiv, mN = h->mN, nN = h->nN;

    // sigma-ordered normalized rows
    uint64_t *len;
    GBLA_TRY(dalloc_t(h, (npiv > mN ? npiv : mN) + 1, &len));
    GBLA_TRY(dalloc_t(h, npiv + 1, &h->ab_ptr));
    GBLA_TRY(dalloc_t(h, mN + 1, &h->cd_ptr));
    GBLA_TRY(dalloc_t(h, npiv + 1, &h->ab_np));
    GBLA_TRY(dalloc_t(h, mN + 1, &h->cd_np));
    k_row_len<<<grid_for(npiv + 1, 256), 256, 0, st>>>(npiv, h->pivot_row, h->row_ptr, len); note_launch();
    GBLA_TRY(exclusive_scan<uint64_t>(h, len, h->ab_ptr, npiv + 1));
    uint64_t tmp64[2];
    GBLA_CUDA_TRY(cudaMemcpyAsync(&tmp64[0], h->ab_ptr + npiv, 8, cudaMemcpyDeviceToHost, st));
    k_row_len<<<grid_for(mN + 1, 256), 256, 0, st>>>(mN, h->nonpivot_row, h->row_ptr, len); note_launch();
    GBLA_TRY(exclusive_scan<uint64_t>(h, len, h->cd_ptr, mN + 1));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&tmp64[1], h->cd_ptr + mN, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->nnz_ab = (int64_t)tmp64[0];
    h->nnz_cd = (int64_t)tmp64[1];
    GBLA_TRY(dalloc_t(h, h->nnz_ab, &h->ab_col));
    GBLA_TRY(dalloc_t(h, h->nnz_ab, &h->ab_val));
    GBLA_TRY(dalloc_t(h, h->nnz_cd, &h->cd_col));
    GBLA_TRY(dalloc_t(h, h->nnz_cd, &h->cd_val));
    if (npiv)
        k_fill_rows<<<grid_for(npiv * 32, 256), 256, 0, st>>>(npiv, npiv, h->pivot_row, h->row_ptr, h->col, h->val,
                                                              h->inv_lead, h->sigma, h->F, h->ab_ptr, h->ab_col,
                                                              h->ab_val, h->ab_np); note_launch();
    if (mN)
        k_fill_rows<<<grid_for(mN * 32, 256), 256, 0, st>>>(mN, npiv, h->nonpivot_row, h->row_ptr, h->col, h->val,
                                                            h->inv_lead, h->sigma, h->F, h->cd_ptr, h->cd_col,
                                                            h->cd_val, h->cd_np); note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());

    // pivot row weights (nnz), used for the Alg 2 op count; the two-row
    // multilines are built on first use (ensure_multilines: INT-pipe path only)
    GBLA_TRY(dalloc_t(h, npiv + 1, &h->ab_w));
    if (npiv) k_row_w<<<grid_for(npiv, 256), 256, 0, st>>>(npiv, h->ab_ptr, h->ab_w); note_launch();

    // targets sorted by sigma(lead): longest first
    GBLA_TRY(dalloc_t(h, mN + 1, &h->order));
    if (mN) {
        uint32_t *keys_out, *it;
        GBLA_TRY(dalloc_t(h, mN, &keys_out));
        GBLA_TRY(dalloc_t(h, mN, &it));
        k_iota<<<grid_for(mN, 256), 256, 0, st>>>(mN, it); note_launch();
        {
            size_t tb = 0;
            GBLA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, h->tlead, keys_out, it, h->order, (int)mN, 0,
                                                          32, st));
            void *t;
            GBLA_TRY(dalloc(h, tb + 16, &t));
            GBLA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(t, tb, h->tlead, keys_out, it, h->order, (int)mN, 0, 32, st));
        }
    }

    // dense D quadrant (the current D until a reduction updates it)
    h->ldD = (nN + 127) / 128 * 128;
    if (h->ldD == 0) h->ldD = 128;
    GBLA_TRY(dalloc_t(h, (size_t)(mN > 0 ? mN : 1) * h->ldD, &h->D));
    GBLA_CUDA_TRY(cudaMemsetAsync(h->D, 0, (size_t)(mN > 0 ? mN : 1) * h->ldD * 2, st));
    if (mN && nN)
        k_densify<<<grid_for(mN * 32, 256), 256, 0, st>>>(mN, h->cd_ptr, h->cd_col, h->cd_val, npiv, n, h->D, h->ldD); note_launch();
    GBLA_TRY(dalloc_t(h, mN + 1, &h->opcount));
    GBLA_CUDA_TRY(cudaMemsetAsync(h->opcount, 0, (mN + 1) * 8, st));
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

// Two-row multilines of A|B, built on first use by the INT-pipe
// kernels (the tensor-core path reads the sigma-ordered rows directly).
gbla_status ensure_multilines(gbla_mat h)
{
    if (h->ml_ptr) return GBLA_OK;
    cudaStream_t st = h->stream;
    const int64_t npiv = h->npiv;
    const int64_t np2 = h->npairs;
    uint64_t tmp64 = 0;
    uint64_t *cnt;
    GBLA_TRY(dalloc_t(h, np2 + 1, &cnt));
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->ml_ptr));
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->ml_np));
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->ml_skip));
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->ml_a01));
    k_ml_count<<<grid_for(np2 + 1, 128), 128, 0, st>>>(np2, npiv, h->ab_ptr, h->ab_col, cnt, h->ml_np, h->ml_skip); note_launch();
    GBLA_TRY(exclusive_scan<uint64_t>(h, cnt, h->ml_ptr, np2 + 1));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&tmp64, h->ml_ptr + np2, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->nslots = (int64_t)tmp64;
    GBLA_TRY(dalloc_t(h, h->nslots, &h->ml_col));
    GBLA_TRY(dalloc_t(h, h->nslots, &h->ml_val));
    if (np2)
        k_ml_fill<<<grid_for(np2, 128), 128, 0, st>>>(np2, npiv, h->ab_ptr, h->ab_col, h->ab_val, h->ml_ptr,
                                                      h->ml_col, h->ml_val, h->ml_a01); note_launch();
    // column runs over the multiline slots
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->mr_ptr));
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->mr_skip));
    GBLA_TRY(dalloc_t(h, np2 + 1, &h->mr_np));
    k_mlr_count<<<grid_for((np2 + 1) * 32, 256), 256, 0, st>>>(np2, h->ml_ptr, h->ml_col, h->ml_skip, h->ml_np, cnt);
    note_launch();
    GBLA_TRY(exclusive_scan<uint64_t>(h, cnt, h->mr_ptr, np2 + 1));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&tmp64, h->mr_ptr + np2, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->nruns = (int64_t)tmp64;
    GBLA_TRY(dalloc_t(h, h->nruns + 1, &h->mr_col));
    GBLA_TRY(dalloc_t(h, h->nruns + 1, &h->mr_len));
    GBLA_TRY(dalloc_t(h, h->nruns + 1, &h->mr_rel));
    if (np2)
        k_mlr_fill<<<grid_for(np2 * 32, 256), 256, 0, st>>>(np2, h->ml_ptr, h->ml_col, h->ml_skip, h->ml_np, h->mr_ptr,
                                                            h->mr_col, h->mr_len, h->mr_rel, h->mr_skip, h->mr_np);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}
