// echelon.cu -- Step 4, fully reduced (reading R13): R = RREF(D)
// by blocked Gauss-Jordan over column panels of width K.
//
// Invariant before panel [c0, c0+K): every row is either a pivot row (its
// pivot column < c0) or ACTIVE, and active rows are zero on all columns < c0
// (a column < c0 is either a pivot column, eliminated from every other row,
// or a column in which no active row was nonzero).  Per panel:
//   K10 k_panel     one CTA scans the active rows in order and builds, in
//                   shared memory, the reduced echelon basis of their panel
//                   slices (incremental: reduce a candidate by the basis; if
//                   nonzero, normalize at its first nonzero column and
//                   eliminate that column from the basis).  It records the
//                   selected rows S, their pivot columns and the transform T
//                   with basis = T * D[S, panel].  It stops early when the
//                   basis has K rows (full rank panel).  The resulting pivot
//                   columns are the canonical ones (the basis is an RREF).
//       k_gather    F[i] = D[i, pivot columns] for every non-selected row
//                   (active AND earlier pivot rows: back elimination), plus
//                   the list of rows with F[i] != 0
//       k_rnew      Rn = T * D[S, c0:]    (new pivot rows, full width)
//   K11 trailing    D[i, c0:] -= F[i] * Rn    (modular GEMM; this file: the
//                   INT-pipe engine; tc_gemm.cu: the tcgen05 engine)
//       k_commit    D[S, c0:] = Rn; rowpiv[S] = pivot columns
// At the end K13 compacts R (rows sorted by pivot column) and pivcol.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace {

constexpr int PK = 64;            // panel width of the INT engine
constexpr unsigned FULL = 0xffffffffu;

struct PanelState {
    uint32_t kp;                  // pivots found in this panel
    uint32_t nrows;               // rows with a nonzero coefficient
    uint32_t sel[PK];             // selected rows
    uint32_t pc[PK];              // absolute pivot columns
    uint16_t T[PK * PK];          // basis = T * D[S, panel]
};

// One CTA, 1024 threads.  Lane l of warp 0 holds panel columns 2l, 2l+1.
__global__ void __launch_bounds__(1024) k_panel(int64_t mN, int64_t nN, int64_t c0, Field F,
                                                const uint16_t *__restrict__ D, int64_t ldD,
                                                uint32_t *__restrict__ rowpiv, PanelState *__restrict__ ps)
{
    __shared__ uint32_t basis[PK][PK];
    __shared__ uint32_t Tm[PK][PK];
    __shared__ uint32_t bpc[PK];
    __shared__ uint32_t bsel[PK];
    __shared__ uint32_t cand[1024];
    __shared__ uint32_t wcount[32];
    __shared__ uint32_t s_ncand, s_nb;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t width = (nN - c0) < PK ? (nN - c0) : PK;
    if (tid == 0) s_nb = 0;
    __syncthreads();
    for (int64_t base = 0; base < mN; base += 1024) {
        // 1. candidates of this chunk, in row order
        int64_t r = base + tid;
        bool cand_ok = false;
        if (r < mN && rowpiv[r] == GBLA_NONE) {
            const uint16_t *row = D + (size_t)r * ldD + c0;
            for (int64_t c = 0; c < width; c++)
                if (row[c]) { cand_ok = true; break; }
        }
        unsigned msk = __ballot_sync(FULL, cand_ok);
        if (lane == 0) wcount[warp] = __popc(msk);
        __syncthreads();
        if (tid == 0) {
            uint32_t s = 0;
            for (int w = 0; w < 32; w++) { uint32_t c = wcount[w]; wcount[w] = s; s += c; }
            s_ncand = s;
        }
        __syncthreads();
        if (cand_ok) cand[wcount[warp] + __popc(msk & ((1u << lane) - 1u))] = (uint32_t)r;
        __syncthreads();
        // 2. warp 0 integrates the candidates
        if (warp == 0) {
            uint32_t nb = s_nb;
            for (uint32_t ci = 0; ci < s_ncand && nb < PK; ci++) {
                const uint32_t rr = cand[ci];
                const uint16_t *row = D + (size_t)rr * ldD + c0;
                uint32_t x0 = (2 * lane < width) ? row[2 * lane] : 0;
                uint32_t x1 = (2 * lane + 1 < width) ? row[2 * lane + 1] : 0;
                uint32_t a0 = (2 * lane == (int)nb) ? 1u : 0u, a1 = (2 * lane + 1 == (int)nb) ? 1u : 0u;
                for (uint32_t b = 0; b < nb; b++) {
                    const uint32_t pcb = bpc[b];
                    uint32_t xv = (pcb & 1) ? x1 : x0;
                    uint32_t f = __shfl_sync(FULL, xv, pcb >> 1);
                    if (f) {
                        const uint32_t nf = F.p - f;
                        x0 = fmod64(x0 + (uint64_t)nf * basis[b][2 * lane], F);
                        x1 = fmod64(x1 + (uint64_t)nf * basis[b][2 * lane + 1], F);
                        a0 = fmod64(a0 + (uint64_t)nf * Tm[b][2 * lane], F);
                        a1 = fmod64(a1 + (uint64_t)nf * Tm[b][2 * lane + 1], F);
                    }
                }
                unsigned nzm = __ballot_sync(FULL, (x0 | x1) != 0);
                if (!nzm) continue;                                   // in the span: dependent
                const int src = __ffs(nzm) - 1;
                uint32_t first0 = __shfl_sync(FULL, x0, src);
                uint32_t first1 = __shfl_sync(FULL, x1, src);
                const uint32_t c = first0 ? 2 * src : 2 * src + 1;
                const uint32_t inv = finv(first0 ? first0 : first1, F);
                x0 = fmul(x0, inv, F); x1 = fmul(x1, inv, F);
                a0 = fmul(a0, inv, F); a1 = fmul(a1, inv, F);
                for (uint32_t b = 0; b < nb; b++) {
                    const uint32_t g = basis[b][c];
                    __syncwarp();
                    if (g) {
                        const uint32_t ng = F.p - g;
                        basis[b][2 * lane] = fmod64(basis[b][2 * lane] + (uint64_t)ng * x0, F);
                        basis[b][2 * lane + 1] = fmod64(basis[b][2 * lane + 1] + (uint64_t)ng * x1, F);
                        Tm[b][2 * lane] = fmod64(Tm[b][2 * lane] + (uint64_t)ng * a0, F);
                        Tm[b][2 * lane + 1] = fmod64(Tm[b][2 * lane + 1] + (uint64_t)ng * a1, F);
                    }
                    __syncwarp();
                }
                basis[nb][2 * lane] = x0; basis[nb][2 * lane + 1] = x1;
                Tm[nb][2 * lane] = a0; Tm[nb][2 * lane + 1] = a1;
                if (lane == 0) { bpc[nb] = c; bsel[nb] = rr; }
                nb++;
                __syncwarp();
            }
            if (lane == 0) s_nb = nb;
        }
        __syncthreads();
        if (s_nb >= PK) break;
    }
    const uint32_t nb = s_nb;
    if (tid == 0) { ps->kp = nb; ps->nrows = 0; }
    for (int i = tid; i < PK * PK; i += blockDim.x) {
        int b = i / PK, s = i % PK;
        ps->T[i] = (b < (int)nb && s < (int)nb) ? (uint16_t)Tm[b][s] : 0;
    }
    if (tid < (int)nb) {
        ps->sel[tid] = bsel[tid];
        ps->pc[tid] = (uint32_t)c0 + bpc[tid];
        rowpiv[bsel[tid]] = (uint32_t)c0 + bpc[tid];    // marks S (pivot col >= c0)
    }
}

// F[i][b] = D[i][pc_b] for rows not selected in this panel; row list of the
// rows with a nonzero coefficient.  One thread per row.
__global__ void k_gather(int64_t mN, int64_t c0, const uint16_t *__restrict__ D, int64_t ldD,
                         const uint32_t *__restrict__ rowpiv, PanelState *__restrict__ ps,
                         uint16_t *__restrict__ Fc, uint32_t *__restrict__ rows)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t kp = ps->kp;
    if (i >= mN || kp == 0) return;
    const uint32_t rp = rowpiv[i];
    if (rp != GBLA_NONE && rp >= (uint64_t)c0) return;   // selected now: becomes Rn
    bool nz = false;
    for (uint32_t b = 0; b < kp; b++) {
        uint16_t v = D[(size_t)i * ldD + ps->pc[b]];
        Fc[(size_t)i * PK + b] = v;
        nz |= v != 0;
    }
    if (nz) {
        uint32_t slot = atomicAdd(&ps->nrows, 1u);
        rows[slot] = (uint32_t)i;
    }
}

// Rn[b][x] = sum_s T[b][s] * D[S_s][c0 + x]
__global__ void k_rnew(int64_t nN, int64_t c0, Field F, const uint16_t *__restrict__ D, int64_t ldD,
                       const PanelState *__restrict__ ps, uint16_t *__restrict__ Rn, int64_t ldR)
{
    const uint32_t kp = ps->kp;
    const uint32_t b = blockIdx.y;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= kp || c0 + x >= nN) return;
    uint64_t acc = 0;
    for (uint32_t s = 0; s < kp; s++) {
        uint32_t t = ps->T[b * PK + s];
        if (t) acc += (uint64_t)t * D[(size_t)ps->sel[s] * ldD + c0 + x];
    }
    Rn[(size_t)b * ldR + x] = (uint16_t)fmod64(acc, F);
}

// INT-pipe trailing update: 32 listed rows x 256 columns per CTA.
__global__ void __launch_bounds__(256) k_trailing_int(int64_t nN, int64_t c0, Field F, uint16_t *__restrict__ D,
                                                      int64_t ldD, const PanelState *__restrict__ ps,
                                                      const uint16_t *__restrict__ Fc,
                                                      const uint32_t *__restrict__ rows,
                                                      const uint16_t *__restrict__ Rn, int64_t ldR,
                                                      unsigned long long *__restrict__ dense_ops)
{
    __shared__ uint32_t sF[32][PK + 1];
    __shared__ uint16_t sR[PK][256];
    const uint32_t kp = ps->kp, nr = ps->nrows;
    const int64_t width = nN - c0;
    const int64_t row0 = (int64_t)blockIdx.y * 32;
    const int64_t x0 = (int64_t)blockIdx.x * 256;
    if (kp == 0 || row0 >= nr || x0 >= width) return;
    const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0)
        atomicAdd(dense_ops, (unsigned long long)nr * kp * width + (unsigned long long)kp * kp * width);
    for (int i = tid; i < 32 * PK; i += 256) {
        int rr = i / PK, b = i % PK;
        sF[rr][b] = (row0 + rr < nr && b < (int)kp) ? Fc[(size_t)rows[row0 + rr] * PK + b] : 0;
    }
    for (int i = tid; i < PK * 256; i += 256) {
        int b = i / 256, x = i % 256;
        sR[b][x] = (b < (int)kp && x0 + x < width) ? Rn[(size_t)b * ldR + x0 + x] : 0;
    }
    __syncthreads();
    uint64_t acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int u = 0; u < 8; u++) acc[a][u] = 0;
    for (uint32_t b = 0; b < kp; b++) {
        uint32_t f[4], r[8];
#pragma unroll
        for (int a = 0; a < 4; a++) f[a] = sF[grp * 4 + a][b];
#pragma unroll
        for (int u = 0; u < 8; u++) r[u] = sR[b][lane + 32 * u];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int u = 0; u < 8; u++) acc[a][u] += (uint64_t)f[a] * r[u];
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int64_t rr = row0 + grp * 4 + a;
        if (rr >= nr) continue;
        uint16_t *drow = D + (size_t)rows[rr] * ldD + c0 + x0;
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int64_t x = lane + 32 * u;
            if (x0 + x < width) {
                uint32_t s = fmod64(acc[a][u], F);
                uint32_t d = drow[x];
                uint32_t v = d >= s ? d - s : d + F.p - s;
                drow[x] = (uint16_t)v;
            }
        }
    }
}

__global__ void k_commit(int64_t nN, int64_t c0, uint16_t *__restrict__ D, int64_t ldD,
                         const PanelState *__restrict__ ps, const uint16_t *__restrict__ Rn, int64_t ldR)
{
    const uint32_t b = blockIdx.y;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= ps->kp || c0 + x >= nN) return;
    D[(size_t)ps->sel[b] * ldD + c0 + x] = Rn[(size_t)b * ldR + x];
}

__global__ void k_reset_rows(PanelState *ps) { ps->nrows = 0; }

// K13: R rows sorted by pivot column.
__global__ void k_mark(int64_t mN, const uint32_t *__restrict__ rowpiv, uint32_t *__restrict__ colrow)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < mN && rowpiv[i] != GBLA_NONE) colrow[rowpiv[i]] = (uint32_t)i;
}
__global__ void k_colflag(int64_t nN, const uint32_t *__restrict__ colrow, uint32_t *__restrict__ flag)
{
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nN) flag[c] = colrow[c] != GBLA_NONE;
    else if (c == nN) flag[c] = 0;
}
__global__ void k_compact(int64_t nN, int64_t cbase, const uint32_t *__restrict__ colrow,
                          const uint32_t *__restrict__ idx, const uint16_t *__restrict__ D, int64_t ldD,
                          uint16_t *__restrict__ R, int64_t ldR, uint32_t *__restrict__ pivcol)
{
    const int64_t c = cbase + blockIdx.y;
    if (c >= nN) return;
    const uint32_t r = colrow[c];
    if (r == GBLA_NONE) return;
    const uint32_t k = idx[c];
    if (threadIdx.x == 0 && blockIdx.x == 0) pivcol[k] = (uint32_t)c;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nN; x += (int64_t)gridDim.x * blockDim.x)
        R[(size_t)k * ldR + x] = D[(size_t)r * ldD + x];
}

}  // namespace

gbla_status echelon_impl(gbla_mat h, uint32_t flags)
{
    cudaStream_t st = h->stream;
    const int64_t mN = h->mN, nN = h->nN, ldD = h->ldD;
    (void)flags;
    uint32_t *rowpiv, *rows, *colrow, *cflag, *cidx;
    uint16_t *Fc, *Rn;
    PanelState *ps;
    unsigned long long *dops;
    const int64_t ldR = ldD;
    GBLA_TRY(dalloc_t(h, mN + 1, &rowpiv));
    GBLA_TRY(dalloc_t(h, mN + 1, &rows));
    GBLA_TRY(dalloc_t(h, (size_t)(mN + 1) * PK, &Fc));
    GBLA_TRY(dalloc_t(h, (size_t)PK * ldR, &Rn));
    GBLA_TRY(dalloc(h, sizeof(PanelState), (void **)&ps));
    GBLA_TRY(dalloc_t(h, 1, &dops));
    GBLA_CUDA_TRY(cudaMemsetAsync(rowpiv, 0xff, (mN + 1) * 4, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(dops, 0, 8, st));
    if (mN > 0 && nN > 0) {
        for (int64_t c0 = 0; c0 < nN; c0 += PK) {
            const int64_t width = nN - c0;
            k_panel<<<1, 1024, 0, st>>>(mN, nN, c0, h->F, h->D, ldD, rowpiv, ps); note_launch();
            k_gather<<<grid_for(mN, 256), 256, 0, st>>>(mN, c0, h->D, ldD, rowpiv, ps, Fc, rows); note_launch();
            k_rnew<<<dim3(grid_for(width, 256), PK), 256, 0, st>>>(nN, c0, h->F, h->D, ldD, ps, Rn, ldR); note_launch();
            dim3 tg(grid_for(width, 256), grid_for(mN, 32));
            k_trailing_int<<<tg, 256, 0, st>>>(nN, c0, h->F, h->D, ldD, ps, Fc, rows, Rn, ldR, dops); note_launch();
            k_commit<<<dim3(grid_for(width, 256), PK), 256, 0, st>>>(nN, c0, h->D, ldD, ps, Rn, ldR); note_launch();
            GBLA_CUDA_TRY(cudaGetLastError());
        }
    }
    // K13: compaction
    GBLA_TRY(dalloc_t(h, nN + 1, &colrow));
    GBLA_TRY(dalloc_t(h, nN + 1, &cflag));
    GBLA_TRY(dalloc_t(h, nN + 1, &cidx));
    GBLA_CUDA_TRY(cudaMemsetAsync(colrow, 0xff, (nN + 1) * 4, st));
    k_mark<<<grid_for(mN, 256), 256, 0, st>>>(mN, rowpiv, colrow); note_launch();
    k_colflag<<<grid_for(nN + 1, 256), 256, 0, st>>>(nN, colrow, cflag); note_launch();
    {
        size_t tb = 0;
        GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, cflag, cidx, (int)(nN + 1), st));
        void *t;
        GBLA_TRY(dalloc(h, tb + 16, &t));
        GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t, tb, cflag, cidx, (int)(nN + 1), st));
    }
    uint32_t rk = 0;
    unsigned long long dv = 0;
    GBLA_CUDA_TRY(cudaMemcpyAsync(&rk, cidx + nN, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(&dv, dops, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->rank = rk;
    h->dense_ops = dv;
    h->ldR = ldD;
    GBLA_TRY(dalloc_t(h, (size_t)(rk > 0 ? rk : 1) * h->ldR, &h->R));
    GBLA_TRY(dalloc_t(h, rk + 1, &h->pivcol));
    if (rk > 0 && nN > 0) {
        const unsigned gx = grid_for(nN, 256) < 8 ? grid_for(nN, 256) : 8;
        for (int64_t cb = 0; cb < nN; cb += 65535) {   // gridDim.y <= 65535
            int64_t cnt = nN - cb < 65535 ? nN - cb : 65535;
            k_compact<<<dim3(gx, (unsigned)cnt), 256, 0, st>>>(nN, cb, colrow, cidx, h->D, ldD, h->R, h->ldR,
                                                               h->pivcol); note_launch();
        }
        GBLA_CUDA_TRY(cudaGetLastError());
    }
    return GBLA_OK;
}
