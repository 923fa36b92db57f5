// echelon.cu -- Step 4, fully reduced (reading R13): R = RREF(D)
// by blocked Gauss-Jordan over column panels of width PK.
//
// Invariant before panel [c0, c0+PK): every row is either a pivot row (its
// pivot column < c0) or ACTIVE, and active rows are zero on all columns < c0
// (a column < c0 is either a pivot column, eliminated from every other row,
// or a column in which no active row was nonzero).  Per panel:
//   K10 k_panel     one CTA (1024 threads) builds, in shared memory, the
//                   reduced echelon basis of the active rows' panel slices:
//                   candidates (active rows with a nonzero slice, in row
//                   order) come in chunks; a chunk is first reduced by the
//                   current basis in parallel (delayed u64 reduction), then
//                   integrated one row at a time: a nonzero row is normalized
//                   at its first nonzero column (inverse table) and that
//                   column is eliminated from the basis and from the rest of
//                   the chunk by the whole CTA.  Each row carries its
//                   transform, so the basis is T * D[S, panel] for the
//                   selected rows S.  The scan stops when the basis has PK
//                   rows.  The basis is an RREF of the panel's row space, so
//                   its pivot columns are the canonical ones.
//       k_gather    F[i] = D[i, pivot columns] for every non-selected row
//                   (active AND earlier pivot rows: back elimination), plus
//                   the list of rows with F[i] != 0
//       Rn          Rn = T * D[S, c0:]    (new pivot rows, full width)
//   K11 trailing    D[i, c0:] -= F[i] * Rn    (modular GEMM)
//       k_commit    D[S, c0:] = Rn; rowpiv[S] = pivot columns
// Engines: GBLA_DENSE_TC (default): PK = 128, Rn and the trailing update on
// tcgen05 (tc_gemm.cu); GBLA_DENSE_INT: PK = 64, both on the INT pipe.
// At the end K13 compacts R (rows sorted by pivot column) and pivcol.
#include <stdio.h>
#include <stdlib.h>

#include <cub/cub.cuh>
#include <vector>

#include "internal.cuh"
#include "tc.cuh"

gbla_status panels_tc2(gbla_mat h, uint32_t *rowpiv, unsigned long long *dops, const uint16_t *invtab);
gbla_status panels_dist(gbla_mat h, uint32_t *rowpiv, unsigned long long *dops, const uint16_t *invtab, int G,
                        int me, bool real);

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int KPT = 128;          // K width of the tensor-core operand planes

template <int PK>
struct PanelState {
    uint32_t kp;                  // pivots found in this panel
    uint32_t nrows;               // rows with a nonzero coefficient
    uint32_t ncand;               // candidate rows scanned by the panel
    uint32_t sel[PK];             // selected rows
    uint32_t pc[PK];              // absolute pivot columns
    uint16_t T[PK * PK];          // basis = T * D[S, panel]
};

// inverse table: inv[a] = a^-1 mod p (inv[0] = 0)
__global__ void k_invtab(Field F, uint16_t *__restrict__ inv)
{
    const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < F.p) inv[a] = a ? (uint16_t)finv(a, F) : 0;
}

template <int PK>
constexpr int panel_smem() { return (2 * PK) * PK * (int)sizeof(uint32_t) + PK * PK * (int)sizeof(uint16_t); }

template <int PK>
__global__ void __launch_bounds__(1024) k_panel(int64_t mN, int64_t nN, int64_t c0, Field F,
                                                const uint16_t *__restrict__ D, int64_t ldD,
                                                uint32_t *__restrict__ rowpiv, PanelState<PK> *__restrict__ ps,
                                                uint8_t *__restrict__ Tlo, uint8_t *__restrict__ Thi,
                                                const uint16_t *__restrict__ invtab,
                                                const uint8_t *__restrict__ cflag,
                                                unsigned long long *__restrict__ trace)
{
    // optional per-panel trace (GBLA_PANEL_TRACE): cycles in scan / load / reduce / integrate,
    // candidates, pivots, chunks
    // (kept in shared memory, updated by thread 0 only: no registers held across the loop)
    __shared__ unsigned long long tr[8];
    __shared__ long long tmark;
    if (trace && threadIdx.x == 0) {
        for (int k = 0; k < 8; k++) tr[k] = 0;
        tmark = clock64();
    }
#define PANEL_LAP(k_)                                                  \
    do {                                                               \
        if (trace && threadIdx.x == 0) { const long long t_ = clock64(); tr[k_] += t_ - tmark; tmark = t_; } \
    } while (0)
    constexpr int CH = PK;             // candidates per chunk
    constexpr int CPL = PK / 32;       // columns per lane
    extern __shared__ uint32_t dsm32[];
    // rows [0, PK): basis; rows [PK, PK + CH): candidates.  Each entry packs the
    // panel value (low 16 bits) and the transform coefficient (high 16 bits).
    uint32_t(*XA)[PK] = reinterpret_cast<uint32_t(*)[PK]>(dsm32);
    uint16_t(*FS)[PK] = reinterpret_cast<uint16_t(*)[PK]>(dsm32 + (PK + CH) * PK);   // [CH][PK] factors
    __shared__ uint32_t bpc[PK], bsel[PK], crow[CH], selfc[CH];
    __shared__ uint32_t brow[PK];      // physical XA row of basis slot b during a chunk
    __shared__ uint32_t skey[CH], perm[CH];
    __shared__ uint32_t Ub[32][33], Wb[32][33];   // block of U and its inverse (back substitution)
    __shared__ uint16_t Gs[PK][32];               // factors of the rows above a block
    __shared__ uint32_t sinv[PK];
    const uint32_t m32 = 0xffffffffu / F.p;   // 32-bit Barrett: v < 2^32 -> v mod p
    auto mod32 = [&](uint32_t v) -> uint32_t {
        const uint32_t r = v - __umulhi(v, m32) * F.p;
        return r >= F.p ? r - F.p : r;
    };
    __shared__ uint32_t wcount[32];
    __shared__ int s_ncand;
    __shared__ long long s_next;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t p = F.p;
    const int64_t width = (nN - c0) < PK ? (nN - c0) : PK;
    if (tid < PK) brow[tid] = tid;
    uint32_t nb = 0, ncand_tot = 0;
    int64_t pos = 0;
    while (nb < (uint32_t)PK && pos < mN) {
        // (1) next chunk of up to CH candidates (k_cand flags), in row order:
        //     scan 1024 rows per round until the chunk is full or the rows run out
        int ncand = 0;
        while (ncand < CH && pos < mN) {
            const int64_t r = pos + tid;
            const bool ok = r < mN && cflag[r] != 0;
            const unsigned msk = __ballot_sync(FULL, ok);
            if (lane == 0) wcount[warp] = __popc(msk);
            __syncthreads();
            if (tid == 0) {
                uint32_t s = 0;
                for (int w = 0; w < 32; w++) { const uint32_t c = wcount[w]; wcount[w] = s; s += c; }
                s_ncand = (ncand + (int)s) < CH ? ncand + (int)s : CH;
                s_next = pos + 1024;
            }
            __syncthreads();
            const uint32_t rank = ncand + wcount[warp] + __popc(msk & ((1u << lane) - 1u));
            if (ok && rank < (uint32_t)CH) crow[rank] = (uint32_t)r;
            if (ok && rank == (uint32_t)CH) s_next = r;      // first candidate not taken
            __syncthreads();
            ncand = s_ncand;
            pos = s_next;
        }
        PANEL_LAP(0);
        if (ncand == 0) continue;
        ncand_tot += ncand;
        if (trace && tid == 0) { tr[4] += ncand; tr[6] += 1; }
        // (2) load the candidates' panel slices
        for (int idx = tid; idx < ncand * PK; idx += 1024) {
            const int ci = idx / PK, k = idx % PK;
            XA[PK + ci][k] = k < width ? D[(size_t)crow[ci] * ldD + c0 + k] : 0;
        }
        if (tid < ncand) selfc[tid] = 1;
        __syncthreads();
        PANEL_LAP(1);
        // (3) reduce the chunk by the current basis (RREF, so each factor is the
        //     candidate's original entry at the basis pivot column)
        if (nb > 0) {
            // snapshot of the factors, then 8-column items (u64 delayed reduction)
            for (int idx = tid; idx < ncand * (int)nb; idx += 1024) {
                const int ci = idx / (int)nb, b = idx % (int)nb;
                FS[ci][b] = (uint16_t)(XA[PK + ci][bpc[b]] & 0xffffu);
            }
            __syncthreads();
            for (int item = tid; item < ncand * (PK / 8); item += 1024) {
                const int ci = item / (PK / 8), g8 = item % (PK / 8);
                uint64_t ax[8], aa[8];
#pragma unroll
                for (int u = 0; u < 8; u++) { ax[u] = XA[PK + ci][g8 * 8 + u] & 0xffffu; aa[u] = 0; }
                for (uint32_t b = 0; b < nb; b++) {
                    const uint32_t f = FS[ci][b];
                    if (!f) continue;
                    const uint64_t nf = p - f;
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const uint32_t v = XA[b][g8 * 8 + u];
                        ax[u] += nf * (v & 0xffffu);
                        aa[u] += nf * (v >> 16);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; u++)
                    XA[PK + ci][g8 * 8 + u] = fmod64(ax[u], F) | (fmod64(aa[u], F) << 16);
            }
            __syncthreads();
        }
        PANEL_LAP(2);
        // (4a) order the chunk by leading column: in a staircase the rest of the
        //      chunk is then zero at each new pivot column (no forward work)
        for (int ci = warp; ci < ncand; ci += 32) {
            bool nz = false;
#pragma unroll
            for (int u = 0; u < CPL; u++) nz |= (XA[PK + ci][lane * CPL + u] & 0xffffu) != 0;
            const unsigned m = __ballot_sync(FULL, nz);
            if (lane == 0) {
                uint32_t key = 0xffffu;
                if (m) {
                    const int src = __ffs(m) - 1;
                    key = src * CPL;
                    while ((XA[PK + ci][key] & 0xffffu) == 0) key++;
                }
                skey[ci] = key;
            }
        }
        __syncthreads();
        if (tid < ncand) {
            const uint32_t kc = skey[tid];
            int rk = 0;
            for (int j = 0; j < ncand; j++) rk += (skey[j] < kc) || (skey[j] == kc && j < tid);
            perm[rk] = tid;
        }
        __syncthreads();
        // (4b) integrate the chunk row by row, in that order
        for (int q = 0; q < ncand && nb < (uint32_t)PK; q++) {
            const int ci = perm[q];
            const uint32_t *cx = XA[PK + ci];
            bool nz = false;
#pragma unroll
            for (int u = 0; u < CPL; u++) nz |= (cx[lane * CPL + u] & 0xffffu) != 0;
            const unsigned nzm = __ballot_sync(FULL, nz);
            if (!nzm) continue;                                  // dependent on the basis
            const int src = __ffs(nzm) - 1;
            uint32_t c = src * CPL;
            while ((cx[c] & 0xffffu) == 0) c++;
            // Forward, fraction-free step (no inverse on the critical path): the
            // pivot row P = candidate ci (pivot value v at column c; its own
            // transform coefficient sc at index nb) joins the basis unreduced,
            // and every remaining candidate R becomes  v*R - g*P,  g = R[c].
            // The basis is reduced and normalized afterwards in blocks (4c).
            const uint32_t v = cx[c] & 0xffffu;
            const uint32_t sc = selfc[ci];
            const int nrows = ncand - q - 1;
            if (tid == 0) {
                // P joins the basis as slot nb (in place; its transform gets sc at index nb)
                XA[PK + ci][nb] = (XA[PK + ci][nb] & 0xffffu) | (sc << 16);
                brow[nb] = PK + ci;
                bpc[nb] = c;
                bsel[nb] = crow[ci];
            }
            for (int rr = warp; rr < nrows; rr += 32) {     // one warp per remaining candidate
                const int cand = perm[q + 1 + rr];
                const uint32_t row = (uint32_t)(PK + cand);
                const uint32_t gl = (lane == (int)(c / CPL)) ? (XA[row][c] & 0xffffu) : 0u;
                const uint32_t g = __shfl_sync(FULL, gl, c / CPL);
                if (!g) continue;
                const uint32_t ng = p - g;
#pragma unroll
                for (int u = 0; u < CPL; u++) {
                    const int k = lane * CPL + u;
                    const uint32_t val = XA[row][k], P = cx[k];
                    const uint32_t pa = (k == (int)nb) ? sc : (P >> 16);
                    const uint32_t x = mod32(mod32(v * (val & 0xffffu)) + ng * (P & 0xffffu));
                    const uint32_t a = mod32(mod32(v * (val >> 16)) + ng * pa);
                    XA[row][k] = x | (a << 16);
                }
                if (lane == 0) selfc[cand] = mod32(v * selfc[cand]);
            }
            __syncthreads();
            nb++;
        }
        PANEL_LAP(3);
        // (4c) compact the basis into slots [0, nb): slot b < nb0 already there
        for (int idx = tid; idx < (int)nb * PK; idx += 1024) {
            const int b = idx / PK, k = idx % PK;
            if (brow[b] != (uint32_t)b) XA[b][k] = XA[brow[b]][k];
        }
        __syncthreads();
        if (tid < (int)nb) brow[tid] = tid;
        // (4d) reduce + normalize the basis, 32-row blocks from the bottom.  U[i][j] =
        //      row_i at pivot column j is upper triangular (old rows: identity on old
        //      pivots; new rows: zero at every earlier pivot).  Per block: W = U_bb^-1
        //      (one warp), block <- W * block, then the block's pivot columns are
        //      eliminated from every row above (u64 delayed reduction, one mod).
        for (int r1 = (int)nb; r1 > 0; r1 -= 32) {
            const int r0 = r1 - 32 > 0 ? r1 - 32 : 0, bs = r1 - r0;
            __syncthreads();
            for (int idx = tid; idx < bs * bs; idx += 1024) {
                const int i = idx / bs, j = idx % bs;
                Ub[i][j] = XA[r0 + i][bpc[r0 + j]] & 0xffffu;
            }
            __syncthreads();
            if (warp == 0) {
                const int j = lane;
                if (j < bs) sinv[j] = invtab[Ub[j][j]];
                __syncwarp();
                if (j < bs) {
                    Wb[j][j] = sinv[j];
                    for (int i = j - 1; i >= 0; i--) {
                        uint64_t acc = 0;
                        for (int k = i + 1; k <= j; k++) acc += (uint64_t)Ub[i][k] * Wb[k][j];
                        Wb[i][j] = fmul(fneg(fmod64(acc, F), F), sinv[i], F);
                    }
                    for (int i = j + 1; i < bs; i++) Wb[i][j] = 0;
                }
            }
            // factors of the rows above at the block's pivot columns (before they change)
            for (int idx = tid; idx < r0 * bs; idx += 1024) {
                const int r = idx / bs, k = idx % bs;
                Gs[r][k] = (uint16_t)(XA[r][bpc[r0 + k]] & 0xffffu);
            }
            __syncthreads();
            // block <- W * block  (items: 4 consecutive columns of one block row)
            static_assert(32 * (PK / 4) <= 1024, "one block-multiply item per thread");
            uint32_t outv[4];
            {
                const int item = tid;
                if (item < bs * (PK / 4)) {
                const int i = item / (PK / 4), k0 = (item % (PK / 4)) * 4;
                uint64_t ax[4] = {0, 0, 0, 0}, aa[4] = {0, 0, 0, 0};
                for (int k = i; k < bs; k++) {
                    const uint64_t w = Wb[i][k];
                    if (!w) continue;
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const uint32_t val = XA[r0 + k][k0 + u];
                        ax[u] += w * (val & 0xffffu);
                        aa[u] += w * (val >> 16);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; u++) outv[u] = fmod64(ax[u], F) | (fmod64(aa[u], F) << 16);
                }
            }
            __syncthreads();
            if (tid < bs * (PK / 4)) {
                const int i = tid / (PK / 4), k0 = (tid % (PK / 4)) * 4;
#pragma unroll
                for (int u = 0; u < 4; u++) XA[r0 + i][k0 + u] = outv[u];
            }
            __syncthreads();
            // rows above: R <- R - sum_k g_k * block_k
            for (int item = tid; item < r0 * (PK / 4); item += 1024) {
                const int r = item / (PK / 4), k0 = (item % (PK / 4)) * 4;
                uint64_t ax[4], aa[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t val = XA[r][k0 + u];
                    ax[u] = val & 0xffffu;
                    aa[u] = val >> 16;
                }
                for (int k = 0; k < bs; k++) {
                    const uint32_t g = Gs[r][k];
                    if (!g) continue;
                    const uint64_t ng = p - g;
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const uint32_t val = XA[r0 + k][k0 + u];
                        ax[u] += ng * (val & 0xffffu);
                        aa[u] += ng * (val >> 16);
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; u++) XA[r][k0 + u] = fmod64(ax[u], F) | (fmod64(aa[u], F) << 16);
            }
        }
        __syncthreads();
        PANEL_LAP(7);
    }
    __syncthreads();
    if (trace && tid == 0) {
        tr[5] = nb;
        unsigned long long *o = trace + (c0 / PK) * 8;
        for (int k = 0; k < 8; k++) o[k] = tr[k];
    }
#undef PANEL_LAP
    if (tid == 0) { ps->kp = nb; ps->nrows = 0; ps->ncand = ncand_tot; }
    for (int i = tid; i < PK * PK; i += blockDim.x) {
        const int b = i / PK, s = i % PK;
        ps->T[i] = (b < (int)nb && s < (int)nb) ? (uint16_t)(XA[b][s] >> 16) : 0;
    }
    if (Tlo) {   // T as one A tile (limb planes, core-matrix layout), zero padded: A operand of the Rn GEMM
        for (int i = tid; i < KPT * KPT; i += blockDim.x) {
            const int b = i / KPT, s = i % KPT;
            const uint16_t v = (b < (int)nb && s < (int)nb && b < PK && s < PK) ? (uint16_t)(XA[b][s] >> 16) : 0;
            const uint32_t o = tc::toff((uint32_t)b, (uint32_t)s);
            Tlo[o] = (uint8_t)(v & 0xff);
            Thi[o] = (uint8_t)(v >> 8);
        }
    }
    if (tid < (int)nb) {
        ps->sel[tid] = bsel[tid];
        ps->pc[tid] = (uint32_t)c0 + bpc[tid];
        rowpiv[bsel[tid]] = (uint32_t)c0 + bpc[tid];    // marks S (pivot col >= c0)
    }
}

// candidate flags of panel [c0, c0+PK): active row with a nonzero slice.
// One thread per row, all slice loads issued together.
template <int PK>
__global__ void k_cand(int64_t mN, int64_t nN, int64_t c0, const uint16_t *__restrict__ D, int64_t ldD,
                       const uint32_t *__restrict__ rowpiv, uint8_t *__restrict__ cflag)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= mN) return;
    bool ok = false;
    if (rowpiv[r] == GBLA_NONE) {
        const uint16_t *row = D + (size_t)r * ldD + c0;
        if (nN - c0 >= PK) {
            uint4 v[PK / 8];
#pragma unroll
            for (int c = 0; c < PK / 8; c++) v[c] = *reinterpret_cast<const uint4 *>(row + 8 * c);
            uint32_t o = 0;
#pragma unroll
            for (int c = 0; c < PK / 8; c++) o |= v[c].x | v[c].y | v[c].z | v[c].w;
            ok = o != 0;
        } else {
            for (int64_t c = 0; c < nN - c0; c++) ok |= row[c] != 0;
        }
    }
    cflag[r] = ok;
}

// F[i][b] = D[i][pc_b] for rows not selected in this panel, compacted to the
// list of rows with a nonzero coefficient.  INT engine: Fc[i][PK] u16 by row;
// TC engine: limb planes by slot, zero padded to KPT.
template <int PK, bool TC>
__global__ void k_gather(int64_t mN, int64_t c0, const uint16_t *__restrict__ D, int64_t ldD,
                         const uint32_t *__restrict__ rowpiv, PanelState<PK> *__restrict__ ps,
                         uint16_t *__restrict__ Fc, uint8_t *__restrict__ Flo, uint8_t *__restrict__ Fhi,
                         uint32_t *__restrict__ rows, int ref)
{
    // one warp per row; lane l holds coefficients b = l*CPL .. l*CPL+CPL-1
    constexpr int CPL = PK / 32;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t kp = ps->kp;
    if (i >= mN || kp == 0) return;
    const uint32_t rp = rowpiv[i];
    if (rp != GBLA_NONE && (rp >= (uint64_t)c0 || ref)) return;   // selected now: becomes Rn (REF: any pivot row)
    const uint16_t *drow = D + (size_t)i * ldD;
    uint16_t v[CPL];
    bool nz = false;
#pragma unroll
    for (int u = 0; u < CPL; u++) {
        const uint32_t b = lane * CPL + u;
        v[u] = b < kp ? drow[ps->pc[b]] : 0;
        nz |= v[u] != 0;
    }
    if (!__any_sync(FULL, nz)) return;
    uint32_t slot = 0;
    if (lane == 0) slot = atomicAdd(&ps->nrows, 1u);
    slot = __shfl_sync(FULL, slot, 0);
    if (lane == 0) rows[slot] = (uint32_t)i;
    if (TC) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int u = 0; u < CPL; u++) {
            lo |= (uint32_t)(v[u] & 0xff) << (8 * u);
            hi |= (uint32_t)(v[u] >> 8) << (8 * u);
        }
        static_assert(!TC || CPL == 4, "TC engine: 4 coefficients per lane");
        // A tiles of the trailing GEMM: 128 slots per tile, core-matrix layout
        const size_t o = (size_t)(slot / 128) * (KPT * 128) + tc::toff(slot % 128, lane * CPL);
        *reinterpret_cast<uint32_t *>(Flo + o) = lo;
        *reinterpret_cast<uint32_t *>(Fhi + o) = hi;
    } else {
#pragma unroll
        for (int u = 0; u < CPL; u++) Fc[(size_t)i * PK + lane * CPL + u] = v[u];
    }
}

// TC engine: transposed limb planes of D[S, c0:]: Bt[x][s] = D[sel_s][c0 + x]
__global__ void k_gather_st(int64_t nN, int64_t c0, const uint16_t *__restrict__ D, int64_t ldD,
                            const PanelState<KPT> *__restrict__ ps, uint8_t *__restrict__ Blo,
                            uint8_t *__restrict__ Bhi)
{
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c0 + x >= nN) return;
    const uint32_t kp = ps->kp;
    {
        const uint32_t s = blockIdx.y * 16;      // one 16-row group of S per grid row
        uint8_t lo[16], hi[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
            const uint16_t v = (s + u < kp) ? D[(size_t)ps->sel[s + u] * ldD + c0 + x] : 0;
            lo[u] = (uint8_t)(v & 0xff);
            hi[u] = (uint8_t)(v >> 8);
        }
        // B tiles of the Rn GEMM: 64 columns per tile, core-matrix layout (K = s)
        const size_t o = (size_t)(x / 64) * (64 * KPT) + tc::toff64((uint32_t)(x % 64), s);
        *reinterpret_cast<uint4 *>(Blo + o) = *reinterpret_cast<uint4 *>(lo);
        *reinterpret_cast<uint4 *>(Bhi + o) = *reinterpret_cast<uint4 *>(hi);
    }
}

// INT engine: Rn[b][x] = sum_s T[b][s] * D[S_s][c0 + x]
template <int PK>
__global__ void k_rnew(int64_t nN, int64_t c0, Field F, const uint16_t *__restrict__ D, int64_t ldD,
                       const PanelState<PK> *__restrict__ ps, uint16_t *__restrict__ Rn, int64_t ldR)
{
    const uint32_t kp = ps->kp;
    const uint32_t b = blockIdx.y;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= kp || c0 + x >= nN) return;
    uint64_t acc = 0;
    for (uint32_t s = 0; s < kp; s++) {
        const uint32_t t = ps->T[b * PK + s];
        if (t) acc += (uint64_t)t * D[(size_t)ps->sel[s] * ldD + c0 + x];
    }
    Rn[(size_t)b * ldR + x] = (uint16_t)fmod64(acc, F);
}

// INT-pipe trailing update: 32 listed rows x 256 columns per CTA (PK = 64).
__global__ void __launch_bounds__(256) k_trailing_int(int64_t nN, int64_t c0, Field F, uint16_t *__restrict__ D,
                                                      int64_t ldD, const PanelState<64> *__restrict__ ps,
                                                      const uint16_t *__restrict__ Fc,
                                                      const uint32_t *__restrict__ rows,
                                                      const uint16_t *__restrict__ Rn, int64_t ldR)
{
    constexpr int PK = 64;
    __shared__ uint32_t sF[32][PK + 1];
    __shared__ uint16_t sR[PK][256];
    const uint32_t kp = ps->kp, nr = ps->nrows;
    const int64_t width = nN - c0;
    const int64_t row0 = (int64_t)blockIdx.y * 32;
    const int64_t x0 = (int64_t)blockIdx.x * 256;
    if (kp == 0 || row0 >= nr || x0 >= width) return;
    const int tid = threadIdx.x, lane = tid & 31, grp = tid >> 5;
    for (int i = tid; i < 32 * PK; i += 256) {
        const int rr = i / PK, b = i % PK;
        sF[rr][b] = (row0 + rr < nr && b < (int)kp) ? Fc[(size_t)rows[row0 + rr] * PK + b] : 0;
    }
    for (int i = tid; i < PK * 256; i += 256) {
        const int b = i / 256, x = i % 256;
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
                const uint32_t s = fmod64(acc[a][u], F);
                const uint32_t d = drow[x];
                drow[x] = (uint16_t)(d >= s ? d - s : d + F.p - s);
            }
        }
    }
}

template <int PK>
__global__ void k_commit(int64_t nN, int64_t c0, uint16_t *__restrict__ D, int64_t ldD,
                         const PanelState<PK> *__restrict__ ps, const uint16_t *__restrict__ Rn, int64_t ldR)
{
    const uint32_t b = blockIdx.y;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= ps->kp || c0 + x >= nN) return;
    D[(size_t)ps->sel[b] * ldD + c0 + x] = Rn[(size_t)b * ldR + x];
}

// algorithmic dense modMACs of the panel: ops[0] += nrows*kp*width (trailing
// update), ops[1] += kp*kp*width (new pivot rows)
template <int PK>
__global__ void k_count(int64_t width, const PanelState<PK> *__restrict__ ps, unsigned long long *__restrict__ ops)
{
    const unsigned long long kp = ps->kp, nr = ps->nrows;
    ops[0] += nr * kp * (unsigned long long)width;
    ops[1] += kp * kp * (unsigned long long)width;
    ops[2] += (unsigned long long)ps->ncand * kp * PK;   // panel RREF: each pivot eliminated from every candidate
    ops[3] += nr * (unsigned long long)width;              // D entries of the trailing update
}

// K13: R rows sorted by pivot column.
__global__ void k_mark(int64_t mN, const uint32_t *__restrict__ rowpiv, uint32_t *__restrict__ colrow)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < mN && rowpiv[i] != GBLA_NONE) colrow[rowpiv[i]] = (uint32_t)i;
}
__global__ void k_colflag(int64_t nN, const uint32_t *__restrict__ colrow, uint32_t *__restrict__ flag)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
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

template <int PK>
gbla_status set_panel_smem()
{
    static unsigned long long done = 0;   // devices done (dev_bit)
    if (!(done & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_panel<PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem<PK>()));
        done |= dev_bit();
    }
    return GBLA_OK;
}

gbla_status panels_int(gbla_mat h, uint32_t *rowpiv, unsigned long long *dops, const uint16_t *invtab)
{
    constexpr int PK = 64;
    cudaStream_t st = h->stream;
    const int64_t mN = h->mN, nN = h->nN, ldD = h->ldD, ldR = h->ldD;
    uint32_t *rows;
    uint16_t *Fc, *Rn;
    PanelState<PK> *ps;
    GBLA_TRY(dalloc_t(h, mN + 1, &rows));
    GBLA_TRY(dalloc_t(h, (size_t)(mN + 1) * PK, &Fc));
    GBLA_TRY(dalloc_t(h, (size_t)PK * ldR, &Rn));
    GBLA_TRY(dalloc(h, sizeof(PanelState<PK>), (void **)&ps));
    GBLA_TRY(set_panel_smem<PK>());
    uint8_t *cflag;
    GBLA_TRY(dalloc_t(h, mN + 1, &cflag));
    for (int64_t c0 = 0; c0 < nN; c0 += PK) {
        const int64_t width = nN - c0;
        k_cand<PK><<<grid_for(mN, 256), 256, 0, st>>>(mN, nN, c0, h->D, ldD, rowpiv, cflag);
        k_panel<PK><<<1, 1024, panel_smem<PK>(), st>>>(mN, nN, c0, h->F, h->D, ldD, rowpiv, ps, nullptr, nullptr,
                                                        invtab, cflag, nullptr);
        note_launch();
        k_gather<PK, false><<<grid_for(mN * 32, 256), 256, 0, st>>>(mN, c0, h->D, ldD, rowpiv, ps, Fc, nullptr, nullptr,
                                                              rows, h->ref_only ? 1 : 0);
        k_rnew<PK><<<dim3(grid_for(width, 256), PK), 256, 0, st>>>(nN, c0, h->F, h->D, ldD, ps, Rn, ldR);
        k_trailing_int<<<dim3(grid_for(width, 256), grid_for(mN, 32)), 256, 0, st>>>(nN, c0, h->F, h->D, ldD, ps,
                                                                                      Fc, rows, Rn, ldR);
        k_commit<PK><<<dim3(grid_for(width, 256), PK), 256, 0, st>>>(nN, c0, h->D, ldD, ps, Rn, ldR);
        k_count<PK><<<1, 1, 0, st>>>(width, ps, dops);
        note_launch(6);
        GBLA_CUDA_TRY(cudaGetLastError());
    }
    return GBLA_OK;
}

}  // namespace

gbla_status bsub_rref(gbla_mat h);   // sparse_tc.cu (K14)

// distinct leading columns of D's rows (warp per row; flag[c] set once, cnt counts first setters)
__global__ void k_lead_distinct(int64_t mN, int64_t nN, const uint16_t *__restrict__ D, int64_t ldD,
                                uint32_t *__restrict__ flag, unsigned int *__restrict__ cnt)
{
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < mN;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint16_t *row = D + (size_t)r * ldD;
        int64_t res = nN;
        for (int64_t base = 0; base < nN && res == nN; base += 32 * 8) {
            int64_t first = nN;
            for (int u = 0; u < 8; u++) {
                const int64_t k = base + lane * 8 + u;
                if (k < nN && row[k] != 0) { first = k; break; }
            }
            const unsigned m = __ballot_sync(0xffffffffu, first < nN);
            if (m) res = __shfl_sync(0xffffffffu, first, __ffs(m) - 1);
        }
        if (lane == 0 && res < nN && atomicExch(&flag[res], 1u) == 0u) atomicAdd(cnt, 1u);
    }
}

// The fully reduced form through a row echelon form and one back substitution (K14, sparse_tc.cu)
// instead of the Gauss-Jordan back elimination inside the panels (GBLA_BACKSUB=0/1 forces it).
// The REF panels touch only rows leading inside each window, so on a staircase D_new (the F4
// shape: c1, c2, c4) the echelon becomes the panel chain plus a triangular solve on the tensor
// cores (c2: 48 ms REF + the solve against 260 ms of Gauss-Jordan).
// Which one: a row echelon form is cheap when the rows of D mostly lead in columns of their own
// (each panel then touches only the few rows colliding in its window); when most rows lead in the
// same few columns (a dense D, c3) the REF does nearly the Gauss-Jordan trailing work and the
// solve comes on top (c3: 153 vs 123 ms).  Rule: the rows lead in at least min(mN, nN) / 4 distinct
// columns (measured fractions: c1 0.63, c2 0.63, c4 0.47 -- REF + solve: c2 437 -> 311 ms, c4 16.96
// -> 14.39 s; c3 0.11).
static gbla_status use_bsub(gbla_mat h, uint32_t flags, bool *out)
{
    *out = false;
    if (flags & (GBLA_ECHELON_REF | GBLA_DENSE_INT)) return GBLA_OK;
    const char *e = getenv("GBLA_BACKSUB");
    if (e) { *out = atoi(e) != 0; return GBLA_OK; }
    if (h->mN < 2 || h->nN < 2) return GBLA_OK;
    cudaStream_t st = h->stream;
    uint32_t *flag;
    unsigned int *cnt;
    GBLA_TRY(dalloc_t(h, h->nN + 1, &flag));
    GBLA_TRY(dalloc_t(h, 1, &cnt));
    GBLA_CUDA_TRY(cudaMemsetAsync(flag, 0, (h->nN + 1) * 4, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(cnt, 0, 4, st));
    const unsigned g = grid_for(h->mN * 32, 256) < 16u * h->ctx->sm_count ? grid_for(h->mN * 32, 256)
                                                                          : 16u * h->ctx->sm_count;
    k_lead_distinct<<<g, 256, 0, st>>>(h->mN, h->nN, h->D, h->ldD, flag, cnt);
    note_launch();
    unsigned int hc = 0;
    GBLA_CUDA_TRY(cudaMemcpyAsync(&hc, cnt, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t lim = h->mN < h->nN ? h->mN : h->nN;
    *out = 4 * (int64_t)hc >= lim;
    if (getenv("GBLA_BSUB_DEBUG"))
        fprintf(stderr, "[gbla echelon] distinct leading columns %u of min(mN, nN) = %lld: %s\n", hc, (long long)lim,
                *out ? "row echelon form + back substitution" : "Gauss-Jordan panels");
    dfree(h, flag);
    return GBLA_OK;
}

gbla_status echelon_impl(gbla_mat h, uint32_t flags)
{
    cudaStream_t st = h->stream;
    h->ref_only = (flags & GBLA_ECHELON_REF) != 0;
    const int64_t mN = h->mN, nN = h->nN, ldD = h->ldD;
    uint32_t *rowpiv, *colrow, *cflag, *cidx;
    uint16_t *invtab;
    unsigned long long *dops;
    GBLA_TRY(dalloc_t(h, mN + 1, &rowpiv));
    GBLA_TRY(dalloc_t(h, 4, &dops));
    GBLA_TRY(dalloc_t(h, 65536, &invtab));
    GBLA_CUDA_TRY(cudaMemsetAsync(rowpiv, 0xff, (mN + 1) * 4, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(dops, 0, 32, st));
    k_invtab<<<grid_for(h->p, 256), 256, 0, st>>>(h->F, invtab);
    note_launch();
    // row-sharded D (multi-GPU, or emulated ranks): the distributed echelon assembles R itself
    const bool real = h->ctx->nccl_comm != nullptr;
    const int G = real ? h->ctx->world : dist_emulated_world();
    if (h->dist_rows && (real || G > 1)) {
        if (flags & GBLA_DENSE_INT) {
            // a row-sharded D holds only this rank's updated rows: the single-GPU INT engine would
            // echelon a partly updated D and give every rank a different (wrong) R
            set_error("gbla_echelon_D: GBLA_DENSE_INT is single-GPU only (D is row-sharded)");
            return GBLA_E_INVAL;
        }
        if (mN > 0 && nN > 0) {
            const gbla_status ds = panels_dist(h, rowpiv, dops, invtab, G, real ? h->ctx->rank : 0, real);
            if (real) GBLA_TRY(dist_check_async(h->ctx));          // a peer's failure first
            GBLA_TRY(ds);
            GBLA_TRY(panel_dev_err(st, "gbla_echelon_D"));
            return tcgemm_dev_err(st, "gbla_echelon_D");
        }
    }
    bool bsub = false;
    if (!(h->dist_rows && (real || G > 1))) GBLA_TRY(use_bsub(h, flags, &bsub));
    if (bsub) h->ref_only = true;            // the panels stop at a row echelon form
    if (mN > 0 && nN > 0) {
        if (flags & GBLA_DENSE_INT) GBLA_TRY(panels_int(h, rowpiv, dops, invtab));
        else GBLA_TRY(panels_tc2(h, rowpiv, dops, invtab));
        GBLA_TRY(panel_dev_err(st, "gbla_echelon_D"));
        GBLA_TRY(tcgemm_dev_err(st, "gbla_echelon_D"));
    }
    // K13: compaction
    GBLA_TRY(dalloc_t(h, nN + 1, &colrow));
    GBLA_TRY(dalloc_t(h, nN + 1, &cflag));
    GBLA_TRY(dalloc_t(h, nN + 1, &cidx));
    GBLA_CUDA_TRY(cudaMemsetAsync(colrow, 0xff, (nN + 1) * 4, st));
    k_mark<<<grid_for(mN, 256), 256, 0, st>>>(mN, rowpiv, colrow);
    k_colflag<<<grid_for(nN + 1, 256), 256, 0, st>>>(nN, colrow, cflag);
    note_launch(2);
    {
        size_t tb = 0;
        GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, cflag, cidx, (int)(nN + 1), st));
        void *t;
        GBLA_TRY(dalloc(h, tb + 16, &t));
        GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t, tb, cflag, cidx, (int)(nN + 1), st));
    }
    uint32_t rk = 0;
    unsigned long long dv[4] = {0, 0, 0, 0};
    GBLA_CUDA_TRY(cudaMemcpyAsync(&rk, cidx + nN, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(dv, dops, 32, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->rank = rk;
    h->dense_ops = dv[0] + dv[1];
    h->kwork[KT_TRAIL] = dv[0];
    h->kwork[KT_RN] = dv[1];
    h->kwork[KT_PANEL] = dv[2];
    h->trail_elems = dv[3];
    h->ldR = ldD;
    GBLA_TRY(dalloc_t(h, (size_t)(rk > 0 ? rk : 1) * h->ldR, &h->R));
    GBLA_TRY(dalloc_t(h, rk + 1, &h->pivcol));
    if (rk > 0 && nN > 0) {
        const unsigned gx = grid_for(nN, 256) < 8 ? grid_for(nN, 256) : 8;
        for (int64_t cb = 0; cb < nN; cb += 65535) {   // gridDim.y <= 65535
            const int64_t cnt = nN - cb < 65535 ? nN - cb : 65535;
            k_compact<<<dim3(gx, (unsigned)cnt), 256, 0, st>>>(nN, cb, colrow, cidx, h->D, ldD, h->R, h->ldR,
                                                               h->pivcol);
            note_launch();
        }
        GBLA_CUDA_TRY(cudaGetLastError());
    }
    if (bsub) {
        h->ref_only = false;
        GBLA_TRY(bsub_rref(h));
        h->dense_ops += h->kwork[KT_BSUB];
    }
    return GBLA_OK;
}
