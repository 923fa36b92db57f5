// panel.cu -- Step 4 (reading R13) on the tensor cores, v2:
// blocked Gauss-Jordan over WIDTH-ADAPTIVE column panels holding up to
// PK = 128 pivots each, so that every trailing update is a K = 128 modular
// GEMM whatever the rank profile of D (a staircase D_new has ~0.4 pivots
// per column, a dense one ~1).
//
// Invariant before the panel starting at column c0 (as in echelon.cu): every
// row is a pivot row (pivot column < c0) or ACTIVE, and active rows are zero
// on all columns < c0.  Per panel (all state on the device; c0 of panel k is
// c1 of panel k-1, so the host never waits between panels):
//   k_lead2    lead[r] = first nonzero column of active row r in [c0, c0+PW)
//   k_panel2   one CTA: the panel width w is the largest w <= PW such that at
//              most PK active rows lead in [c0, c0+w) ("wide" mode: those
//              rows are the candidates, so at most PK pivots); if more than
//              PK rows lead in [c0, c0+128) the panel is [c0, c0+128) and
//              candidates come in chunks ("dense" mode, stop at w pivots).
//              The candidates' panel slices are reduced by the basis, then
//              put in echelon form by parallel ROUNDS: every row finds its
//              leading column, one row per column becomes a head (normalized,
//              established heads first) and eliminates that column from the
//              rows that share it; rounds repeat until all leading columns
//              differ.  A blocked back substitution (32-row blocks, the
//              unit-triangular block inverse by repeated squaring) makes the
//              basis reduced.  Every row carries its coefficients over the
//              candidates (E), so basis = T * D[S, panel] for the selected
//              rows S.
//   k_gather2  F[i] = D[i, pivot columns] for every other row (active rows
//              and earlier pivot rows: back elimination), rows with F != 0
//   K11        Rn = T * D[S, c0:] and D[rows, c0:] -= F * Rn (tc_gemm.cu)
//   k_commit2  D[S, c0:] = Rn, op counts
// The basis of a panel is the RREF of the active rows restricted to
// [c0, c0+w), so its pivot columns are the canonical ones and R is unique.
#include <stdio.h>
#include <stdlib.h>

#include <functional>
#include <utility>
#include <vector>

#include <cub/cub.cuh>

#include "internal.cuh"
#include "tc.cuh"

GBLA_DEV_ERR_UNIT(panel_dev_err)

namespace {

// launch with programmatic dependent launch (the kernel calls pdl_trigger / pdl_wait): its launch
// overlaps the tail of the previous kernel of the stream
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr unsigned FULL = 0xffffffffu;
constexpr int PK = 128;                 // pivots per panel = K of the trailing GEMM
constexpr int PW = 512;                 // widest panel (columns)
constexpr int LDX = PW + PK + 8;        // row of the store: values [0, PW) | coefficients [PW, PW+PK) | pad
                                        // (1296-byte rows: consecutive rows start 4 banks apart)
constexpr int FSLD = PK + 8;            // row stride of the factor snapshot / U (same reason)
constexpr int NT = 1024;                // threads of k_panel2
constexpr uint32_t NONE16 = 0xffffffffu;

struct P2State {
    int64_t c0, c1;                     // panel columns [c0, c1)
    uint32_t kp;                        // pivots
    uint32_t nrows;                     // rows (slots) of the trailing update
    uint32_t ntouch;                    // of which rows with a nonzero coefficient (the op counts)
    uint32_t ncand;                     // candidates integrated
    uint32_t ready;                     // epoch: sel / pc / kp / c0 / c1 / rowpiv marks are published
    uint32_t sel[PK];                   // selected rows (D row ids), pivot order of T
    uint32_t pc[PK];                    // absolute pivot columns
};

constexpr int P2_SMEM = PK * LDX * 2 + PK * FSLD * 2;   // row store + factor snapshot (196 KB)

// Where the panel reads its rows.  Single GPU: all rows of D, window at column c0.
// Distributed echelon: the candidates gathered from every rank (their window slices,
// leads and D row ids), the global lead histogram, and the owner map (rowpiv is only
// marked for this rank's rows).
struct PanelSrc {
    const uint16_t *D;          // row r, window column k at D[r * ldD + (gathered ? 0 : c0) + k]
    int64_t ldD;
    int64_t nrows;
    const uint32_t *lead;       // [nrows] window-relative leading column, NONE if not active
    const uint32_t *rid;        // [nrows] D row id (NULL: identity)
    const uint32_t *ghist;      // [PW] global lead counts (NULL: counted here)
    const uint8_t *owner;       // [mN] rank of each D row (NULL: every row is local)
    int me;
    int gathered;
    int cap;                    // wide panels: at most cap (<= PK) rows lead inside the window
    int walign;                 // panel widths a multiple of this (32 if 0; 64 with deferred updates)
};

// panels per super-panel of deferred trailing updates (GBLA_SP = 1..4).  Default: 4 when D is
// large (the trailing updates are HBM / epilogue bound: c2, c3, c4), else 1 (c1: the panel chain
// is the critical path and the per-panel update is hidden behind it; fix-ups would lengthen it).
static int sp_panels(int64_t mN, int64_t nN, bool ref)
{
    const char *e = getenv("GBLA_SP");
    // a row echelon form (no back elimination) touches only the rows leading inside each window:
    // the prefix rows of a super-panel flush would be zero-factor work (c2: 247 vs 48 ms)
    const int g = e ? atoi(e) : (!ref && (double)mN * (double)nN >= 4e8 ? 4 : 1);
    return g < 1 ? 1 : g > 4 ? 4 : g;
}

// candidates per wide panel (GBLA_PANEL_CAP, default PK): fewer pivots per panel shorten the
// panel factorization (quadratic in them) but add panels
static int panel_cap()
{
    const char *e = getenv("GBLA_PANEL_CAP");
    const int c = e ? atoi(e) : PK;
    return c >= 16 && c <= PK ? c : PK;
}


__device__ __forceinline__ uint32_t mod32(uint32_t v, uint32_t p, uint32_t m32)
{
    const uint32_t r = v - __umulhi(v, m32) * p;
    return r >= p ? r - p : r;
}

__device__ __forceinline__ void ld8(const uint16_t *s, uint32_t (&v)[8])
{
    const uint4 q = *reinterpret_cast<const uint4 *>(s);
    v[0] = q.x & 0xffffu; v[1] = q.x >> 16; v[2] = q.y & 0xffffu; v[3] = q.y >> 16;
    v[4] = q.z & 0xffffu; v[5] = q.z >> 16; v[6] = q.w & 0xffffu; v[7] = q.w >> 16;
}
__device__ __forceinline__ void st8(uint16_t *s, const uint32_t (&v)[8])
{
    *reinterpret_cast<uint4 *>(s) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                               v[6] | (v[7] << 16));
}

// lead[r] = first nonzero column of active row r in [c0, c0 + PW) relative to c0, else NONE.
// One warp per row, 8 columns (16 bytes) per lane per step.
// Row echelon form (srow != NULL: rows sorted by their initial leading column skey, D in place):
// a row's lead only moves right, so only the rows with skey < c0 + PW can lead in the window;
// the others keep lead NONE (set once before the first panel) and are not read.
__global__ void k_lead2(int64_t mN, int64_t nN, const uint16_t *__restrict__ D, int64_t ldD,
                        const uint32_t *__restrict__ rowpiv, const P2State *__restrict__ prev,
                        uint32_t *__restrict__ lead, const uint8_t *__restrict__ owner, int me,
                        const uint32_t *__restrict__ srow = nullptr, const uint32_t *__restrict__ skey = nullptr)
{
    tc::pdl_trigger();
    tc::pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t c0 = prev->c1;
    int64_t nrow = mN;
    if (srow) {
        __shared__ uint32_t s_n;
        if (threadIdx.x == 0) {
            const int64_t c = c0 + PW;
            int64_t lo = 0, hi = mN;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)skey[mid] < c) lo = mid + 1;
                else hi = mid;
            }
            s_n = (uint32_t)lo;
        }
        __syncthreads();
        nrow = s_n;
    }
    for (int64_t ri = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ri < nrow;
         ri += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = srow ? (int64_t)srow[ri] : ri;
    if (owner && owner[r] != me) continue;                 // another rank's row
    uint32_t res = NONE16;
    if (rowpiv[r] == GBLA_NONE && c0 < nN) {
        const int64_t wmax = nN - c0 < PW ? nN - c0 : PW;
        const uint16_t *row = D + (size_t)r * ldD + c0;
        const bool vec = (((size_t)r * ldD + c0) & 7) == 0;  // c0 is a multiple of 32 but at the last panel
        for (int64_t base = 0; base < wmax && res == NONE16; base += 256) {
            const int64_t k0 = base + lane * 8;
            uint32_t first = NONE16;
            if (vec && k0 + 8 <= wmax) {
                const uint4 q = __ldcg(reinterpret_cast<const uint4 *>(row + k0));
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
                uint32_t m = 0;
#pragma unroll
                for (int j = 0; j < 4; j++) m |= ((w[j] & 0xffffu) ? 1u : 0u) << (2 * j) | ((w[j] >> 16) ? 2u : 0u) << (2 * j);
                if (m) first = (uint32_t)k0 + __ffs(m) - 1;
            } else {
                for (int u = 0; u < 8; u++) {
                    const int64_t k = k0 + u;
                    if (k < wmax && row[k] != 0) { first = (uint32_t)k; break; }
                }
            }
            const unsigned m = __ballot_sync(FULL, first != NONE16);
            if (m) res = __shfl_sync(FULL, first, __ffs(m) - 1);
        }
    }
    if (lane == 0) lead[r] = res;
    }
}

// ---- warp-level tensor-core helpers (mma.sync m16n8k32, u8 x u8 -> s32) for the panel's small
// modular products: u16 residues are split into limbs (lo, hi bytes) and a product is
// 2^16 HH + 2^8 (HL + LH) + LL.  Fragment layouts: PTX ISA, mma.m16n8k32 (.u8).
namespace tcs {
__device__ __forceinline__ void mma_u8(uint32_t (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2])
{
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void split4(uint2 v, uint32_t &lo, uint32_t &hi)
{
    lo = __byte_perm(v.x, v.y, 0x6420);
    hi = __byte_perm(v.x, v.y, 0x7531);
}
// A (16 x 32, row-major u16 M with row stride ld): rows r0 + g (+8), columns k0 + 4 t (+16)
__device__ __forceinline__ void frag_a(const uint16_t *M, int ld, int r0, int k0, uint32_t (&lo)[4], uint32_t (&hi)[4])
{
    const int g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
    const uint16_t *p0 = M + (size_t)(r0 + g) * ld + k0 + 4 * t, *p1 = p0 + 8 * (size_t)ld;
    split4(*reinterpret_cast<const uint2 *>(p0), lo[0], hi[0]);
    split4(*reinterpret_cast<const uint2 *>(p1), lo[1], hi[1]);
    split4(*reinterpret_cast<const uint2 *>(p0 + 16), lo[2], hi[2]);
    split4(*reinterpret_cast<const uint2 *>(p1 + 16), lo[3], hi[3]);
}
// B (32 x 8, given transposed: BT row n holds column n, K contiguous): column n0 + g, K k0 + 4 t (+16)
__device__ __forceinline__ void frag_b(const uint16_t *BT, int ld, int n0, int k0, uint32_t (&lo)[2], uint32_t (&hi)[2])
{
    const int g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
    const uint16_t *q = BT + (size_t)(n0 + g) * ld + k0 + 4 * t;
    split4(*reinterpret_cast<const uint2 *>(q), lo[0], hi[0]);
    split4(*reinterpret_cast<const uint2 *>(q + 16), lo[1], hi[1]);
}
// as frag_b on the panel's rotated T^t (row c of BT at X + c * ld, K entry k at (k + 8 (c & 15)) mod 128)
__device__ __forceinline__ void frag_b_rot(const uint16_t *X, int ld, int n0, int k0, uint32_t (&lo)[2], uint32_t (&hi)[2])
{
    const int g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
    const int c = n0 + g;
    const uint16_t *row = X + (size_t)c * ld;
    const int rot = 8 * (c & 15);
    split4(*reinterpret_cast<const uint2 *>(row + ((k0 + 4 * t + rot) & 127)), lo[0], hi[0]);
    split4(*reinterpret_cast<const uint2 *>(row + ((k0 + 16 + 4 * t + rot) & 127)), lo[1], hi[1]);
}
}  // namespace tcs

// Dense chunk echelon form by a blocked LU: column blocks of 32 inside the
// window (ldv <= 128).  Phase F: pivot steps (one barrier each, smallest (lead, row) key) on a
// copy V of the block's columns of the candidate rows, cross-multiplied (row <- v_h row - f head)
// and tracked against the block-start rows Y:  row_r = sigma_r Y_r + sum_j L[r][j] Y_{p_j}.
// Phase U: the columns right of the block and the coefficients get that update at once,
//     X[r][x] = sigma_r Y[r][x] + (L Y_p)[r][x]   (mma.sync m16n8k32 u8 limbs, K = 32),
// the block's columns are V.  Heads are never written again in the chunk (LU: no elimination
// above pivots here; the chunk's back substitution follows).  Returns the pivot steps taken.
// Scratch (dense mode: the value columns >= 128 are unused): V at 128, L at 160, the snapshot
// Y_p^t at 192 (virtual column n -> row n & 127, offset 32 (n >> 7)) of every store row.
__device__ int blocked_lu(uint16_t *X, uint32_t *cstat, uint32_t *clead, uint32_t p, uint32_t m32, const Field &F,
                          int ldv)
{
    __shared__ uint32_t sig[PK];
    __shared__ uint32_t prow[32];
    __shared__ uint32_t wbest[2][32];      // per-warp bids, double-buffered by step parity
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#define BV(q_, j_) X[(q_) * LDX + 128 + (j_)]
#define BL(q_, j_) X[(q_) * LDX + 160 + (j_)]
    // phase F layout: thread = (store row r = tid / 8, lane group gl = tid % 8); it holds the row's
    // block columns 4 gl .. 4 gl + 3 (v) and transform columns 4 gl .. (l) in registers, and
    // publishes them to BV / BL after every change (the next pivot row is read from there)
    const int r = tid >> 3, gl = tid & 7, c4 = 4 * gl;
    const unsigned gmask = 0xffu << (lane & 24);
    int slot = 0, nsteps = 0;
    for (int cb = 0; cb < ldv; cb += 32) {
        const bool loaded = cstat[r] != 0;
        bool fr = cstat[r] == 1;                               // free candidate row
        uint32_t v[4], l[4] = {0, 0, 0, 0}, sg = 1;
        {
            const uint2 q = *reinterpret_cast<const uint2 *>(&X[r * LDX + cb + c4]);
            v[0] = q.x & 0xffffu; v[1] = q.x >> 16; v[2] = q.y & 0xffffu; v[3] = q.y >> 16;
            *reinterpret_cast<uint2 *>(&BV(r, c4)) = q;
            *reinterpret_cast<uint2 *>(&BL(r, c4)) = make_uint2(0, 0);
            if (gl == 0) sig[r] = 1;
        }
        __syncthreads();
        int kj = 0;
        for (;;) {                                                             // phase F
            nsteps++;
            uint32_t ld = NONE16;                                  // the row's lead in the block (group min)
            if (fr) {
#pragma unroll
                for (int i = 3; i >= 0; i--) if (v[i]) ld = (uint32_t)(c4 + i);
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {                      // all lanes: no divergent shuffles
                const uint32_t y = __shfl_xor_sync(FULL, ld, o);
                ld = y < ld ? y : ld;
            }
            uint32_t key = ld != NONE16 ? ((ld << 7) | (uint32_t)r) : NONE16;
            key = __reduce_min_sync(FULL, key);
            if (lane == 0) wbest[slot][warp] = key;              // one slot per warp: no atomics
            __syncthreads();
            key = __reduce_min_sync(FULL, wbest[slot][lane]);
            slot ^= 1;
            if (key == NONE16) break;
            const int c = (int)(key >> 7);
            const int hq = (int)(key & 127u);
            if (r == hq) {
                fr = false;
                if (gl == 0) { cstat[r] = 2; clead[r] = (uint32_t)(cb + c); }
            } else if (fr) {
                const uint32_t src = (uint32_t)((lane & 24) | (c >> 2)), ci = (uint32_t)(c & 3);
                const uint32_t mine = ci == 0 ? v[0] : ci == 1 ? v[1] : ci == 2 ? v[2] : v[3];
                const uint32_t f = __shfl_sync(gmask, mine, src, 32);
                if (f) {
                    const uint32_t vh = BV(hq, c), nf = p - f;
                    const uint2 pv = *reinterpret_cast<const uint2 *>(&BV(hq, c4));
                    const uint2 pl = *reinterpret_cast<const uint2 *>(&BL(hq, c4));
                    const uint32_t pvv[4] = {pv.x & 0xffffu, pv.x >> 16, pv.y & 0xffffu, pv.y >> 16};
                    const uint32_t plv[4] = {pl.x & 0xffffu, pl.x >> 16, pl.y & 0xffffu, pl.y >> 16};
                    const uint32_t sh = sig[hq];
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        v[i] = mod32(mod32(vh * v[i], p, m32) + nf * pvv[i], p, m32);
                        const int j = c4 + i;
                        if (j < kj) l[i] = mod32(mod32(vh * l[i], p, m32) + nf * plv[i], p, m32);
                        else if (j == kj) l[i] = mod32(nf * sh, p, m32);
                    }
                    sg = mod32(vh * sg, p, m32);
                    *reinterpret_cast<uint2 *>(&BV(r, c4)) = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
                    *reinterpret_cast<uint2 *>(&BL(r, c4)) = make_uint2(l[0] | (l[1] << 16), l[2] | (l[3] << 16));
                    if (gl == 0) sig[r] = sg;
                }
            }
            if (tid == 0) prow[kj] = (uint32_t)hq;
            kj++;
            if (kj == 32) {                         // the block is full: every column has a pivot
                __syncthreads();
                break;
            }
        }
        (void)loaded;
        // phase U: block columns = V; the rest of the window and the coefficients by one K = 32 product
        if (kj > 0) {
            const int nv = ldv - cb - 32, nvc = nv + PK;
            for (int idx = tid; idx < PK * 32; idx += NT) {
                const int q = idx >> 5, j = idx & 31;
                if (cstat[q] != 0) X[q * LDX + cb + j] = BV(q, j);
            }
            for (int idx = tid; idx < nvc * 32; idx += NT) {       // snapshot Y_p^t (zero beyond kj)
                const int n = idx >> 5, k = idx & 31;
                const int col = n < nv ? cb + 32 + n : PW + (n - nv);
                X[(n & 127) * LDX + 192 + 32 * (n >> 7) + k] = k < kj ? X[prow[k] * LDX + col] : (uint16_t)0;
            }
            __syncthreads();
            const int g = lane >> 2, t4 = lane & 3;
            const int ntile = 8 * (nvc / 8);
            for (int tile = warp; tile < ntile; tile += 32) {
                const int mt = tile & 7, n0 = (tile >> 3) * 8;
                const int r0 = 16 * mt;
                uint32_t hh[4] = {0, 0, 0, 0}, xx[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
                uint32_t alo[4], ahi[4], blo[2], bhi[2];
                tcs::frag_a(&BL(0, 0), LDX, r0, 0, alo, ahi);
                tcs::frag_b(X + 192 + 32 * (n0 >> 7), LDX, n0 & 127, 0, blo, bhi);
                tcs::mma_u8(hh, ahi, bhi);
                tcs::mma_u8(xx, ahi, blo);
                tcs::mma_u8(ll, alo, blo);
                tcs::mma_u8(xx, alo, bhi);
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int r = r0 + g + ((e >> 1) << 3), n = n0 + 2 * t4 + (e & 1);
                    if (cstat[r] == 0) continue;
                    const int col = n < nv ? cb + 32 + n : PW + (n - nv);
                    const uint32_t z = fmod_limbs(hh[e], xx[e], ll[e], F);
                    uint16_t *y = &X[r * LDX + col];
                    *y = (uint16_t)mod32(mod32(sig[r] * *y, p, m32) + z, p, m32);
                }
            }
            __syncthreads();
        }
    }
#undef BV
#undef BL
    return nsteps;
}

// Inverse W of a unit upper triangular 32 x 32 matrix U (entries beyond bs: identity),
// by doubling block sizes: with the diagonal blocks of size s already inverted,
// each aligned 2s-block [[A, B], [0, C]] gets its off-diagonal block -A^-1 B C^-1.
// Five levels, two products each, all threads; U is left unchanged.
__device__ void unit_upper_inverse(const uint32_t (*U)[33], uint32_t (*W)[33], uint32_t (*Q)[33], const Field &F)
{
    const int tid = threadIdx.x, i = tid >> 5, j = tid & 31;
    W[i][j] = (i == j) ? 1u : 0u;
    __syncthreads();
    for (int s = 1; s < 32; s <<= 1) {
        const int ne = 16 * s;                  // (32 / 2s) pairs x s^2 entries
        int q = 0, r = 0, c = 0, base = 0;
        if (tid < ne) {
            q = tid / (s * s);
            r = (tid / s) % s;
            c = tid % s;
            base = q * 2 * s;
            uint64_t acc = 0;                   // (B C^-1)[r][c]
            for (int k = 0; k <= c; k++) acc += (uint64_t)U[base + r][base + s + k] * W[base + s + k][base + s + c];
            Q[base + r][base + s + c] = fmod64(acc, F);
        }
        __syncthreads();
        if (tid < ne) {
            uint64_t acc = 0;                   // (A^-1 (B C^-1))[r][c]
            for (int k = r; k < s; k++) acc += (uint64_t)W[base + r][base + k] * Q[base + k][base + s + c];
            const uint32_t z = fmod64(acc, F);
            W[base + r][base + s + c] = z ? F.p - z : 0;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(NT, 1) k_panel2(int64_t nN, Field F, PanelSrc src, uint32_t *__restrict__ rowpiv,
                                                   const P2State *__restrict__ prev, P2State *__restrict__ cur,
                                                   uint8_t *__restrict__ Tlo, uint8_t *__restrict__ Thi,
                                                   const uint16_t *__restrict__ invtab,
                                                   unsigned long long *__restrict__ trace, uint32_t epoch)
{
    extern __shared__ __align__(16) uint16_t X[];          // [PK][LDX] row store
    uint16_t(*FS)[FSLD] = reinterpret_cast<uint16_t(*)[FSLD]>(X + PK * LDX);   // factor snapshot
    __shared__ uint32_t hist[PW + 1];       // lead histogram -> prefix; reused as column -> head key
    __shared__ uint32_t crow[PK];           // D row of each physical row of the store
    __shared__ uint32_t clead[PK];          // leading column of each physical row (chunk rounds)
    __shared__ uint32_t cstat[PK];          // 0 free, 1 candidate, 2 head (this chunk), 3 basis
    __shared__ uint32_t bphys[PK];          // physical row of basis slot b (slots sorted by pivot per chunk)
    __shared__ uint32_t bpc[PK];            // pivot column (window-relative) of basis slot b
    __shared__ uint32_t freel[PK];
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t Ub[32][33], Rb[32][33], Qb[32][33];
    constexpr int CLMAX = 1024;
    __shared__ uint32_t clist[CLMAX];        // rows leading inside the window (wide-mode candidates)
    __shared__ uint32_t hinv[PK];            // inverse of each head's leading value (wide mode)
    __shared__ uint32_t hmap[PW];            // rounds: column -> established head of this chunk
    __shared__ uint32_t s_u[8];
    __shared__ uint32_t s_hbits[PW / 32];     // leading columns of the chunk's heads
    __shared__ long long s_pos;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t p = F.p;
    const uint32_t m32 = 0xffffffffu / p;
    const int64_t c0 = prev->c1;
    const int64_t mN = src.nrows;
    const uint32_t *__restrict__ lead = src.lead;
    const uint16_t *__restrict__ D = src.D;
    const int64_t ldD = src.ldD;
    const int64_t coff = src.gathered ? 0 : c0;           // column of window column 0 in D
    bool published = false;                                // S / pivots published early (wide mode)
    // optional trace (GBLA_PANEL_TRACE): cycles per phase, accumulated over panels by thread 0
    // (laps kept in shared memory and flushed once at the end: a global read-modify-write per lap
    // would add its own latency to the next lap)
    __shared__ unsigned long long s_tr[18];
    if (trace && tid < 18) s_tr[tid] = 0;
    long long t_mark = trace ? clock64() : 0;
#define P2_LAP(k_)                                                                        \
    do {                                                                                  \
        if (trace && tid == 0) { const long long t_ = clock64(); s_tr[k_] += t_ - t_mark; t_mark = t_; } \
    } while (0)
    int64_t wmax = nN - c0;
    if (wmax > PW) wmax = PW;
    if (wmax <= 0) {
        if (tid == 0) {
            cur->c0 = c0; cur->c1 = c0; cur->kp = 0; cur->nrows = 0; cur->ntouch = 0; cur->ncand = 0;
            if (epoch) {
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&cur->ready), "r"(epoch) : "memory");
            }
        }
        return;
    }
    // ---- 1. width from the lead histogram
    for (int k = tid; k <= PW; k += NT) hist[k] = 0;
    if (tid == 0) s_u[5] = 0;
    __syncthreads();
    for (int64_t r0 = 0; r0 < mN; r0 += 8 * NT) {           // 8 loads in flight per thread
        uint32_t l8[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int64_t r = r0 + u * NT + tid;
            l8[u] = r < mN ? __ldcg(lead + r) : NONE16;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const uint32_t l = l8[u];
            if (l < (uint64_t)wmax) {
                if (!src.ghist) atomicAdd(&hist[l], 1u);
                const uint32_t q = atomicAdd(&s_u[5], 1u);
                if (q < (uint32_t)CLMAX) clist[q] = (uint32_t)(r0 + u * NT + tid);
            }
        }
    }
    if (src.ghist)
        for (int k = tid; k < wmax; k += NT) hist[k] = src.ghist[k];
    __syncthreads();
    {   // exclusive prefix over hist[0..PW] (threads 0..PW-1 own one entry each; PW <= NT)
        const uint32_t v = tid < PW ? hist[tid] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = wsum[lane], z = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, z, o);
                if (lane >= o) z += y;
            }
            wsum[lane] = z - w;
        }
        __syncthreads();
        const uint32_t excl = x - v + wsum[warp];
        __syncthreads();
        if (tid < PW) hist[tid] = excl;
        if (tid == PW - 1) hist[PW] = excl + v;
        __syncthreads();
    }
    // hist[c] = number of active rows leading in [c0, c0 + c)
    const int64_t w128 = wmax < 128 ? wmax : 128;
    if (tid == 0) { s_u[0] = (uint32_t)w128; s_u[1] = 0; }
    __syncthreads();
    const bool dense = hist[w128] > (uint32_t)PK;
    if (!dense) {
        // widest w with <= PK candidates; a multiple of 32 (c0 stays 64-byte aligned for the
        // GEMM epilogue's vector path; 64 with deferred updates: column tiles of every panel
        // line up) unless the panel reaches the last column
        const int64_t wa = src.walign > 0 ? src.walign - 1 : 31;
        for (int64_t c = w128 + tid; c <= wmax; c += NT)
            if (hist[c] <= (uint32_t)src.cap && (c == wmax || (c & wa) == 0)) atomicMax(&s_u[0], (uint32_t)c);
    }
    __syncthreads();
    const int width = (int)s_u[0];
    P2_LAP(0);
    const int ldv = (width + 31) & ~31;          // value columns kept (multiple of 32)
    static_assert(32 * (128 / 8 + PK / 8) <= NT, "dense-mode block multiply: one item per thread");
    const int cpl = ldv / 32;                    // value columns per lane
    const uint32_t target = dense ? (uint32_t)width : (uint32_t)PK;   // stop when nb reaches it
    for (int k = tid; k < PK; k += NT) cstat[k] = 0;
    __syncthreads();

    // ---- 2. chunks of candidates (rows with lead < width), in row order
    uint32_t nb = 0, ncand_tot = 0;
    int64_t pos = 0;
    while (nb < target && pos < mN) {
        // free physical rows
        if (warp == 0) {
            uint32_t base = 0;
            for (int q0 = 0; q0 < PK; q0 += 32) {
                const bool fr = cstat[q0 + lane] == 0;
                const unsigned m = __ballot_sync(FULL, fr);
                if (fr) freel[base + __popc(m & ((1u << lane) - 1u))] = q0 + lane;
                base += __popc(m);
            }
            if (lane == 0) s_u[2] = base;
        }
        __syncthreads();
        const uint32_t nfree = s_u[2];
        // collect up to nfree candidates from pos on
        int ncand = 0;
        if (!dense && s_u[5] <= (uint32_t)CLMAX) {
            // wide mode: the candidates (<= PK) are in the window list; take them in row order
            const int ncl = (int)s_u[5];
            const int t = tid;
            const uint32_t lt = t < ncl ? lead[clist[t]] : NONE16;
            const bool ok = lt < (uint32_t)width;
            const unsigned msk = __ballot_sync(FULL, ok);
            if (lane == 0) wsum[warp] = __popc(msk);
            __syncthreads();
            if (warp == 0) {                         // exclusive scan of the warp counts
                const uint32_t c = wsum[lane];
                uint32_t x = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= o) x += y;
                }
                wsum[lane] = x - c;
                if (lane == 31) s_u[3] = x;
            }
            __syncthreads();
            if (ok) {                                // clead: rows, hinv: their leads (scratch)
                const uint32_t at = wsum[warp] + __popc(msk & ((1u << lane) - 1u));
                clead[at] = clist[t];
                hinv[at] = lt;
            }
            __syncthreads();
            ncand = (int)s_u[3];
            {   // order by (lead, row): physical ~ pivot order; rank counted by 8 threads per candidate
                const int ct = tid >> 3, part = tid & 7;
                const bool mine = ct < ncand;
                const uint64_t kr = mine ? ((uint64_t)hinv[ct] << 32) | clead[ct] : 0;
                int rk = 0;
                if (mine)
                    for (int j = part; j < ncand; j += 8) rk += (((uint64_t)hinv[j] << 32) | clead[j]) < kr;
                rk += __shfl_xor_sync(FULL, rk, 1);
                rk += __shfl_xor_sync(FULL, rk, 2);
                rk += __shfl_xor_sync(FULL, rk, 4);
                if (mine && part == 0) {
                    crow[freel[rk]] = clead[ct];
                    cstat[freel[rk]] = 1;
                }
            }
            pos = mN;
            __syncthreads();
        }
        while (ncand < (int)nfree && pos < mN) {
            const int64_t r = pos + tid;
            const bool ok = r < mN && lead[r] < (uint32_t)width;
            const unsigned msk = __ballot_sync(FULL, ok);
            if (lane == 0) wsum[warp] = __popc(msk);
            __syncthreads();
            if (tid == 0) {
                uint32_t s = 0;
                for (int w = 0; w < 32; w++) { const uint32_t c = wsum[w]; wsum[w] = s; s += c; }
                s_u[3] = (ncand + (int)s) < (int)nfree ? ncand + s : nfree;
                s_pos = pos + NT;
            }
            __syncthreads();
            const uint32_t rk = ncand + wsum[warp] + __popc(msk & ((1u << lane) - 1u));
            if (ok && rk < nfree) { crow[freel[rk]] = (uint32_t)r; cstat[freel[rk]] = 1; }
            if (ok && rk == nfree) s_pos = r;            // first candidate not taken
            __syncthreads();
            ncand = (int)s_u[3];
            pos = s_pos;
        }
        if (ncand == 0) break;
        ncand_tot += ncand;
        P2_LAP(1);
        // (a) load the chunk: values D[r, c0 + k], coefficients = unit vector at the physical row
        {
            const bool vec = ((coff & 7) == 0) && ((ldD & 7) == 0);
            const int gv = ldv / 8;                   // 8-column groups of values
            for (int idx = tid; idx < ncand * gv; idx += NT) {
                const int ci = idx / gv, g = idx % gv;
                const uint32_t q = freel[ci];
                const uint16_t *srow = D + (size_t)crow[q] * ldD + coff + 8 * g;
                uint4 v;
                if (vec && 8 * g + 8 <= width) {
                    v = *reinterpret_cast<const uint4 *>(srow);
                } else {
                    uint16_t t[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) t[u] = (8 * g + u < width) ? srow[u] : 0;
                    v = *reinterpret_cast<uint4 *>(t);
                }
                *reinterpret_cast<uint4 *>(X + q * LDX + 8 * g) = v;
            }
            for (int idx = tid; idx < ncand * (PK / 8); idx += NT) {    // E = unit vectors, 8 per store
                const int ci = idx / (PK / 8), k8 = (idx % (PK / 8)) * 8;
                const uint32_t q = freel[ci];
                uint4 z = make_uint4(0, 0, 0, 0);
                if ((int)(q & ~7u) == k8) reinterpret_cast<uint16_t *>(&z)[q & 7] = 1;
                *reinterpret_cast<uint4 *>(&X[q * LDX + PW + k8]) = z;
            }
        }
        __syncthreads();
        P2_LAP(2);
        // (b) reduce the chunk by the basis (RREF: the factor is the entry at the basis pivot)
        if (nb > 0) {
            for (int idx = tid; idx < ncand * (int)nb; idx += NT) {
                const int ci = idx / nb, b = idx % nb;
                FS[ci][b] = X[freel[ci] * LDX + bpc[b]];
            }
            __syncthreads();
            const int ng = (ldv + PK) / 8;                 // 8-column groups of values and coefficients
            for (int item = tid; item < ncand * ng; item += NT) {
                const int ci = item / ng, g = item % ng;
                const int k0 = g * 8 < ldv ? g * 8 : PW + (g * 8 - ldv);
                uint16_t *xr = X + freel[ci] * LDX + k0;
                uint32_t v8[8];
                ld8(xr, v8);
                uint64_t acc[8];
#pragma unroll
                for (int u = 0; u < 8; u++) acc[u] = v8[u];
                for (uint32_t b = 0; b < nb; b++) {
                    const uint32_t f = FS[ci][b];
                    if (!f) continue;
                    const uint64_t nf = p - f;
                    ld8(X + bphys[b] * LDX + k0, v8);
#pragma unroll
                    for (int u = 0; u < 8; u++) acc[u] += nf * v8[u];
                }
#pragma unroll
                for (int u = 0; u < 8; u++) v8[u] = fmod64(acc[u], F);
                st8(xr, v8);
            }
            __syncthreads();
        }
        P2_LAP(3);
        // (c) echelon form of the chunk: parallel rounds (staircase panels: many distinct leads)
        //     or pivot steps (dense panels: the rounds would elect one head per round)
        if (!dense) {
            // Two block barriers per round: (c1) every remaining candidate (warp per row) finds
            // its leading column from a cursor (leads only move right) and, while an established
            // head owns it, eliminates it (heads are fixed: no block sync); then it bids for its
            // column (atomicMin of its physical row in this round's election buffer) and prefetches
            // 1 / its leading value.  (c2) the winner of every column becomes a head; the other
            // buffer is cleared for the next round.
            uint32_t *elect[2] = {hist, clist};      // clist is dead once the candidates are loaded
            // Each round walks a compact list of the still-open candidates (the losers of the last
            // election), so the warps share them evenly.  An elimination updates value columns in
            // pairs (32-bit words) and finds the row's next leading column on the way; coefficient
            // columns are updated only in the 32-column chunks where the head's coefficients are
            // nonzero (emask: E starts as unit vectors and a row's chunks grow by its heads').
            __shared__ uint32_t alist[2][PK];
            __shared__ uint32_t s_nact[2];
            __shared__ uint8_t emask[PK];
            for (int k = tid; k < width; k += NT) { hmap[k] = NONE16; hist[k] = NONE16; clist[k] = NONE16; }
            for (int ci = tid; ci < ncand; ci += NT) {
                const uint32_t q = freel[ci];
                clead[q] = 0;
                alist[0][ci] = q;
                emask[q] = nb == 0 ? (uint8_t)(1u << (q >> 5)) : (uint8_t)0xf;
            }
            if (tid == 0) { s_nact[0] = (uint32_t)ncand; s_nact[1] = 0; }
            __syncthreads();
            for (int round = 0;; round++) {
                if (trace && tid == 0) s_tr[8] += 1;
                uint32_t *hb = elect[round & 1];
                const uint32_t *al = alist[round & 1];
                const int nact = (int)s_nact[round & 1];
                // 1 / leading value of every bidder: loaded now, consumed by the election (the
                // table read's latency is not waited for per candidate)
                uint32_t pend[PK / 32];
#pragma unroll
                for (int j = 0; j < PK / 32; j++) {
                    const int ci = warp + 32 * j;
                    pend[j] = 0;
                    if (ci >= nact) continue;
                    const uint32_t q = al[ci];
                    uint16_t *xr = X + q * LDX;
                    uint32_t ld = NONE16;
                    for (int base = (int)(clead[q] & ~31u); base < ldv; base += 32) {
                        const unsigned m = __ballot_sync(FULL, xr[base + lane] != 0);
                        if (m) { ld = base + __ffs(m) - 1; break; }
                    }
                    uint32_t em = emask[q];
                    for (;;) {
                        if (ld == NONE16) {                       // dependent: zero on the panel
                            __syncwarp();
                            if (lane == 0) { cstat[q] = 0; clead[q] = NONE16; }
                            break;
                        }
                        const uint32_t hq = hmap[ld];
                        if (hq == NONE16) {
                            __syncwarp();
                            if (lane == 0) {
                                clead[q] = ld;
                                emask[q] = (uint8_t)em;
                                atomicMin(&hb[ld], q);
                                pend[j] = __ldg(invtab + xr[ld]);
                            }
                            break;
                        }
                        const uint16_t *hr = X + hq * LDX;
                        // dense mode: heads are normalized; wide mode: scale by the head's inverse
                        const uint32_t gl = dense ? xr[ld] : mod32(xr[ld] * hinv[hq], p, m32);
                        const uint32_t ng = gl ? p - gl : 0;
                        __syncwarp();
                        uint32_t nl = NONE16;
                        for (int k0 = (int)(ld & ~31u); k0 < ldv; k0 += 64) {
                            const int k = k0 + 2 * lane;
                            uint32_t lo = 0, hi = 0;
                            if (k < ldv) {
                                const uint32_t xv = *reinterpret_cast<const uint32_t *>(xr + k);
                                const uint32_t hv = *reinterpret_cast<const uint32_t *>(hr + k);
                                lo = mod32((xv & 0xffffu) + ng * (hv & 0xffffu), p, m32);
                                hi = mod32((xv >> 16) + ng * (hv >> 16), p, m32);
                                *reinterpret_cast<uint32_t *>(xr + k) = lo | (hi << 16);
                            }
                            if (nl == NONE16) {
                                const unsigned m = __ballot_sync(FULL, (lo | hi) != 0);
                                if (m) {
                                    const int j = __ffs(m) - 1;
                                    nl = (uint32_t)(k0 + 2 * j) + __shfl_sync(FULL, lo == 0 ? 1u : 0u, j);
                                }
                            }
                        }
                        const uint32_t hm = emask[hq];
#pragma unroll
                        for (int c = 0; c < PK / 32; c++)
                            if ((hm >> c) & 1u) {
                                const int k = PW + 32 * c + lane;
                                xr[k] = (uint16_t)mod32(xr[k] + ng * hr[k], p, m32);
                            }
                        em |= hm;
                        ld = nl;
                        __syncwarp();
                    }
                    __syncwarp();
                }
                __syncthreads();
                P2_LAP(3);
                uint32_t *nl_ = alist[(round + 1) & 1];
#pragma unroll
                for (int j = 0; j < PK / 32; j++) {
                    const int ci = warp + 32 * j;
                    if (ci >= nact) continue;
                    const uint32_t q = al[ci];
                    if (cstat[q] != 1) continue;
                    if (hb[clead[q]] != q) {                     // eliminated next round
                        if (lane == 0) nl_[atomicAdd(&s_nact[(round + 1) & 1], 1u)] = q;
                        continue;
                    }
                    __syncwarp();
                    if (lane == 0) { cstat[q] = 2; hmap[clead[q]] = q; hinv[q] = pend[j]; }
                    if (dense) {                                          // normalized heads
                        uint16_t *xr = X + q * LDX;
                        const uint32_t iv = __shfl_sync(FULL, pend[j], 0);
                        for (int k = (clead[q] & ~31u) + lane; k < ldv; k += 32) xr[k] = (uint16_t)mod32(iv * xr[k], p, m32);
                        for (int k = lane; k < PK; k += 32) xr[PW + k] = (uint16_t)mod32(iv * xr[PW + k], p, m32);
                    }
                    __syncwarp();
                }
                uint32_t *ob = elect[(round + 1) & 1];
                for (int k = tid; k < width; k += NT) ob[k] = NONE16;
                if (tid == 0) s_nact[round & 1] = 0;
                __syncthreads();
                P2_LAP(4);
                if (s_nact[(round + 1) & 1] == 0) break;
            }
        } else {
            // (c) echelon form of the chunk by pivot steps, ONE block barrier per pivot.  Every
            //     candidate (warp-owned, <= 4 per warp) finds its leading column (from a cursor: leads
            //     only move right); the smallest (lead, physical row) key becomes the next head, and
            //     every other candidate with a nonzero f at that column is cross-eliminated,
            //         row <- v_h * row - f * head           (v_h = the head's leading value),
            //     i.e. replaced by a nonzero multiple of its reduced form: no inverse on the chain,
            //     and E (the coefficients) follows the row, so row = E * candidates still holds.  A
            //     head is never written again, so reading it needs no barrier beyond the one that
            //     elected it.  Keys rotate over three slots (a slot is reset two steps after use).
            {
                __shared__ uint32_t skey[3];
                __shared__ uint32_t skey2[2][32];
                if (tid < 3) skey[tid] = NONE16;
                for (int ci = tid; ci < ncand; ci += NT) clead[freel[ci]] = 0;
                __syncthreads();
                int slot = 0, nsteps = 0;
                const bool blocked = ldv <= 128;
                if (blocked) {
                    nsteps = blocked_lu(X, cstat, clead, p, m32, F, ldv);
                } else for (;;) {
                    nsteps++;
                    uint32_t best = NONE16;
                    for (int ci = warp; ci < ncand; ci += 32) {
                        const uint32_t q = freel[ci];
                        if (cstat[q] != 1) continue;
                        const uint16_t *xr = X + q * LDX;
                        uint32_t ld = NONE16;
                        for (int base = (int)(clead[q] & ~31u); base < ldv; base += 32) {
                            const unsigned m = __ballot_sync(FULL, xr[base + lane] != 0);
                            if (m) { ld = base + __ffs(m) - 1; break; }
                        }
                        __syncwarp();
                        if (ld == NONE16) {                       // dependent: zero on the panel
                            if (lane == 0) { cstat[q] = 0; clead[q] = NONE16; }
                        } else {
                            if (lane == 0) clead[q] = ld;
                            const uint32_t key = (ld << 7) | q;
                            best = key < best ? key : best;
                        }
                        __syncwarp();
                    }
                    if (lane == 0) skey2[slot][warp] = best;              // one slot per warp: no atomics
                    __syncthreads();
                    const uint32_t key = __reduce_min_sync(FULL, skey2[slot][lane]);
                    slot ^= 1;
                    if (key == NONE16) break;
                    const uint32_t c = key >> 7, hq = key & 127u;
                    const uint16_t *hr = X + hq * LDX;
                    const uint32_t vh = hr[c];
                    for (int ci = warp; ci < ncand; ci += 32) {
                        const uint32_t q = freel[ci];
                        if (cstat[q] != 1) continue;
                        if (q == hq) {                            // the new head (owned by this warp)
                            __syncwarp();
                            if (lane == 0) cstat[q] = 2;
                            __syncwarp();
                            continue;
                        }
                        uint16_t *xr = X + q * LDX;
                        const uint32_t f = xr[c];
                        __syncwarp();
                        if (!f) continue;
                        const uint32_t nf = p - f;
                        for (int k = (int)(c & ~31u) + lane; k < ldv; k += 32)
                            xr[k] = (uint16_t)mod32(mod32(vh * xr[k], p, m32) + nf * hr[k], p, m32);
                        for (int k = lane; k < PK; k += 32)
                            xr[PW + k] = (uint16_t)mod32(mod32(vh * xr[PW + k], p, m32) + nf * hr[PW + k], p, m32);
                        __syncwarp();
                    }
                }
                if (trace && tid == 0) s_tr[8] += nsteps;
                P2_LAP(3);
                // heads: 1 / leading value (wide mode keeps the row), or normalized rows (dense mode)
                for (int ci = warp; ci < ncand; ci += 32) {
                    const uint32_t q = freel[ci];
                    if (cstat[q] != 2) continue;
                    uint16_t *xr = X + q * LDX;
                    const uint32_t iv = invtab[xr[clead[q]]];
                    __syncwarp();
                    if (!dense) {
                        if (lane == 0) hinv[q] = iv;
                        continue;
                    }
                    for (int k = (clead[q] & ~31u) + lane; k < ldv; k += 32) xr[k] = (uint16_t)mod32(iv * xr[k], p, m32);
                    for (int k = lane; k < PK; k += 32) xr[PW + k] = (uint16_t)mod32(iv * xr[PW + k], p, m32);
                    __syncwarp();
                }
                __syncthreads();
                P2_LAP(4);
            }
        }
        // (d) the chunk's heads, sorted by leading column, become basis slots nb .. nb+h-1
        //     (heads have distinct leading columns: rank = heads left of it, from a column bitmap)
        if (tid < PW / 32) s_hbits[tid] = 0;
        __syncthreads();
        const bool is_head = tid < ncand && cstat[freel[tid]] == 2;
        const uint32_t hq_ = is_head ? freel[tid] : 0, hc_ = is_head ? clead[hq_] : 0;
        if (is_head) atomicOr(&s_hbits[hc_ >> 5], 1u << (hc_ & 31));
        const uint32_t h = (uint32_t)__syncthreads_count(is_head);
        if (is_head) {
            uint32_t rk = __popc(s_hbits[hc_ >> 5] & ((1u << (hc_ & 31)) - 1u));
            for (uint32_t w = 0; w < (hc_ >> 5); w++) rk += __popc(s_hbits[w]);
            bphys[nb + rk] = hq_;
            bpc[nb + rk] = hc_;
        }
        __syncthreads();
        const uint32_t nb0 = nb;
        // dead rows are free again (their coefficient columns are zero in every head)
        for (int ci = tid; ci < ncand; ci += NT) {
            const uint32_t q = freel[ci];
            if (cstat[q] == 1 || cstat[q] == 0) cstat[q] = 0;
            else if (cstat[q] == 2) cstat[q] = 3;
        }
        nb = nb0 + h;
        __syncthreads();
        // (e) back substitution over the new slots, 32-slot blocks from the bottom.  With U = the
        //     basis at its pivot columns (unit upper triangular among the new slots, whose rows
        //     are zero left of their pivots): block <- W block (W = inverse of the block's diagonal
        //     part of U), then every slot above (older slots and new slots above the block) -=
        //     its entries at the block's pivots * block.  A slot's entries at the pivots of other
        //     blocks never change (block rows are zero there), so G is read from the rows as they
        //     are.  Dense mode reduces values and coefficients (later chunks are reduced by the
        //     basis); wide mode (one chunk) only needs the coefficients: T = U^-1 E.
        P2_LAP(4);
        if (!dense) {
            if (epoch) {
                // the pivots are final: publish S, the pivot columns and the window so that the F
                // gather of the next step (k_gather2, waiting on `ready`) overlaps the T solve
                if (tid < (int)nb) {
                    const uint32_t rr = crow[bphys[tid]];
                    const uint32_t r = src.rid ? src.rid[rr] : rr;
                    cur->sel[tid] = r;
                    cur->pc[tid] = (uint32_t)(c0 + bpc[tid]);
                    if (!src.owner || src.owner[r] == src.me) rowpiv[r] = (uint32_t)(c0 + bpc[tid]);
                }
                if (tid == 0) {
                    cur->c0 = c0;
                    cur->c1 = c0 + width;
                    cur->kp = nb;
                    cur->nrows = 0;
                    cur->ntouch = 0;
                    cur->ncand = ncand_tot;
                }
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&cur->ready), "r"(epoch) : "memory");
                }
                published = true;
            }
            // Wide mode (one chunk, nb0 = 0): heads h_b (pivot order, not normalized) with
            // coefficients E_b.  U[b][b'] = h_b[pc_b'] / h_b[pc_b] is unit upper triangular and the
            // RREF basis is W (h_b / h_b[pc_b]) with W = U^-1, so T = W E', E'_b = E_b / h_b[pc_b].
            // W by doubling block sizes (128 x 128, entries beyond nb: identity), then T with the
            // zero entries of E' skipped (E' is nearly diagonal on a staircase).  The value rows
            // are dead now: W and Q live in their first 512 bytes.
            // T = U^-1 E' by a blocked back substitution over 32-slot row blocks, bottom up:
            //     T_I = W_II (E'_I - U_{I,>I} T_{>I}),   W_II = (U_II)^-1,
            // the two products of every block on the warp-level tensor cores (mma.sync m16n8k32
            // u8 -> s32 on the limbs of the u16 residues: HH, HL + LH, LL, each <= 128 * 255^2 * 2
            // < 2^31; S = 2^16 HH + 2^8 X + LL < 2^40 reduced once), one m16n8 output tile per
            // warp.  W_II by doubling inside the four diagonal blocks.  T and the residual are
            // kept transposed (slot-major, so the B fragments are 8-byte loads); the value rows
            // are dead now and hold them.
            // (rows >= nb of U, and rows / columns >= nb of E', only reach outputs that are dropped)
            uint16_t(*U)[FSLD] = FS;
            for (int idx = tid; idx < (int)nb * PK; idx += NT) {
                const int b = idx >> 7, b2 = idx & (PK - 1);
                uint32_t v = (b == b2) ? 1u : 0u;
                if (b2 > b && b2 < (int)nb) v = mod32(X[bphys[b] * LDX + bpc[b2]] * hinv[bphys[b]], p, m32);
                U[b][b2] = (uint16_t)v;
            }
            __syncthreads();
#define TT(c_, k_) X[(c_) * LDX + (((k_) + 8 * ((c_) & 15)) & (PK - 1))]   // T^t: slot c, row k (rows rotated: no bank conflicts)
#define RT(c_, k_) X[(c_) * LDX + PK + (k_)]          // residual of the block, transposed (k < 32)
#define WD(i_, j_) X[(i_) * LDX + PK + 32 + (j_)]     // W_II: row 32 I + i, column j < 32
#define QD(i_, j_) X[(i_) * LDX + PK + 64 + (j_)]     // doubling scratch
#define EP(b_, c_) X[(b_) * LDX + PK + 96 + (((c_) + 8 * ((b_) & 15)) & (PK - 1))]   // E' (rotated rows)
            for (int idx = tid; idx < PK * (PK / 8); idx += NT) {   // T^t = 0 (K padding beyond nb)
                const int c = idx >> 4, k8 = (idx & 15) * 8;
                *reinterpret_cast<uint4 *>(&TT(c, k8)) = make_uint4(0, 0, 0, 0);
            }
            for (int idx = tid; idx < PK * 32; idx += NT) {
                const int i = idx >> 5, j = idx & 31;
                WD(i, j) = (uint16_t)((i & 31) == j ? 1 : 0);
            }
            for (int idx = tid; idx < (int)nb * PK; idx += NT) {   // E'[b][c] = E[phys b][phys c] / h_b[pc_b]
                const int b = idx >> 7, c = idx & (PK - 1);
                uint32_t v = 0;
                if (c < (int)nb) {
                    const uint32_t qb = bphys[b];
                    v = mod32(X[qb * LDX + PW + bphys[c]] * hinv[qb], p, m32);
                }
                EP(b, c) = (uint16_t)v;
            }
            __syncthreads();
            P2_LAP(13);
            // W_II: levels s = 1 .. 16; every aligned 2s-block [[A, B], [0, C]] of a diagonal block
            // gets Q = B C^-1, then -A^-1 Q (64 s items per step, one per thread at s = 16)
            for (int sl = 0; sl < 5; sl++) {
                const int sz = 1 << sl;
                const int items = 64 * sz;
                for (int it = tid; it < items; it += NT) {
                    const int c = it & (sz - 1), r = (it >> sl) & (sz - 1), q = it >> (2 * sl);   // q: pair over 128 rows
                    const int base = q * 2 * sz, lb = base & 31;
                    uint64_t acc = 0;
                    for (int k = 0; k <= c; k++)
                        acc += (uint64_t)U[base + r][base + sz + k] * WD(base + sz + k, lb + sz + c);
                    QD(base + r, lb + sz + c) = (uint16_t)fmod64(acc, F);
                }
                __syncthreads();
                for (int it = tid; it < items; it += NT) {
                    const int c = it & (sz - 1), r = (it >> sl) & (sz - 1), q = it >> (2 * sl);
                    const int base = q * 2 * sz, lb = base & 31;
                    uint64_t acc = 0;
                    for (int k = r; k < sz; k++) acc += (uint64_t)WD(base + r, lb + k) * QD(base + k, lb + sz + c);
                    const uint32_t z = fmod64(acc, F);
                    WD(base + r, lb + sz + c) = (uint16_t)(z ? p - z : 0);
                }
                __syncthreads();
            }
            P2_LAP(14);
            {
                const int g = lane >> 2, t4 = lane & 3;
                const int mt = warp >> 4, n0 = (warp & 15) * 8;      // this warp's m16n8 tile of the block
                const int nblk = ((int)nb + 31) >> 5;
                for (int I = nblk - 1; I >= 0; I--) {
                    const int r0 = 32 * I + 16 * mt;
                    // R_I = E'_I - U_{I,>I} T_{>I}
                    uint32_t hh[4] = {0, 0, 0, 0}, xx[4] = {0, 0, 0, 0}, ll[4] = {0, 0, 0, 0};
                    for (int k0 = 32 * (I + 1); k0 < (int)nb; k0 += 32) {
                        uint32_t alo[4], ahi[4], blo[2], bhi[2];
                        tcs::frag_a(&U[0][0], FSLD, r0, k0, alo, ahi);
                        tcs::frag_b_rot(X, LDX, n0, k0, blo, bhi);
                        tcs::mma_u8(hh, ahi, bhi);
                        tcs::mma_u8(xx, ahi, blo);
                        tcs::mma_u8(ll, alo, blo);
                        tcs::mma_u8(xx, alo, bhi);
                    }
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int row = r0 + g + ((e >> 1) << 3), col = n0 + 2 * t4 + (e & 1);
                        const uint32_t z = fmod_limbs(hh[e], xx[e], ll[e], F);
                        const uint32_t ev = EP(row, col);
                        RT(col, row - 32 * I) = (uint16_t)(ev >= z ? ev - z : ev + p - z);
                    }
                    __syncthreads();
                    // T_I = W_II R_I
#pragma unroll
                    for (int e = 0; e < 4; e++) { hh[e] = 0; xx[e] = 0; ll[e] = 0; }
                    {
                        uint32_t alo[4], ahi[4], blo[2], bhi[2];
                        tcs::frag_a(&WD(0, 0), LDX, r0, 0, alo, ahi);
                        tcs::frag_b(&RT(0, 0), LDX, n0, 0, blo, bhi);
                        tcs::mma_u8(hh, ahi, bhi);
                        tcs::mma_u8(xx, ahi, blo);
                        tcs::mma_u8(ll, alo, blo);
                        tcs::mma_u8(xx, alo, bhi);
                    }
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int row = r0 + g + ((e >> 1) << 3), col = n0 + 2 * t4 + (e & 1);
                        const uint32_t z = fmod_limbs(hh[e], xx[e], ll[e], F);
                        TT(col, row) = (uint16_t)(row < (int)nb ? z : 0u);
                    }
                    __syncthreads();
                }
            }
            P2_LAP(16);
            // the T tile (limb planes, K index = slot): 4 consecutive K entries per 4-byte store;
            // consecutive lanes take consecutive rows bb (one row of T^t: conflict-free)
            for (int idx = tid; idx < PK * PK / 4; idx += NT) {
                const int bb = idx & (PK - 1), l0 = (idx >> 7) * 4;
                uint32_t lo = 0, hi = 0;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t x = (bb < (int)nb && l0 + u < (int)nb) ? TT(l0 + u, bb) : 0u;
                    lo |= (x & 0xffu) << (8 * u);
                    hi |= (x >> 8) << (8 * u);
                }
                const uint32_t o = tc::toff((uint32_t)bb, (uint32_t)l0);
                *reinterpret_cast<uint32_t *>(Tlo + o) = lo;
                *reinterpret_cast<uint32_t *>(Thi + o) = hi;
            }
#undef TT
#undef RT
#undef WD
#undef QD
#undef EP
            P2_LAP(15);
            break;
        }
        const int gv = dense ? ldv / 8 : 0;      // value groups updated
        const int ng = gv + PK / 8;              // + coefficient groups
        for (int r1 = (int)nb; r1 > (int)nb0; r1 -= 32) {
            const int r0 = r1 - 32 > (int)nb0 ? r1 - 32 : (int)nb0, bs = r1 - r0;
            {
                const int i = tid >> 5, j = tid & 31;
                Ub[i][j] = (i < bs && j < bs) ? X[bphys[r0 + i] * LDX + bpc[r0 + j]] : (i == j ? 1u : 0u);
            }
            for (int idx = tid; idx < r0 * bs; idx += NT) {
                const int r = idx / bs, k = idx % bs;
                FS[r][k] = X[bphys[r] * LDX + bpc[r0 + k]];
            }
            __syncthreads();
            P2_LAP(13);
            unit_upper_inverse(Ub, Rb, Qb, F);     // Rb = block inverse
            P2_LAP(14);
            // block <- W * block (read everything, then write); bs * ng <= 32 * 32 = NT items
            if (tid == 0) s_u[6] = 0;
            uint32_t outv[8];
            const int item = tid;
            if (item < bs * ng) {
                const int i = item / ng, g = item % ng;
                const int k0 = g < gv ? g * 8 : PW + (g - gv) * 8;
                uint64_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int k = i; k < bs; k++) {
                    const uint64_t w = Rb[i][k];
                    if (!w) continue;
                    uint32_t v8[8];
                    ld8(X + bphys[r0 + k] * LDX + k0, v8);
#pragma unroll
                    for (int u = 0; u < 8; u++) acc[u] += w * v8[u];
                }
#pragma unroll
                for (int u = 0; u < 8; u++) outv[u] = fmod64(acc[u], F);
            }
            __syncthreads();
            if (item < bs * ng) {
                const int i = item / ng, g = item % ng;
                const int k0 = g < gv ? g * 8 : PW + (g - gv) * 8;
                st8(X + bphys[r0 + i] * LDX + k0, outv);
                if (outv[0] | outv[1] | outv[2] | outv[3] | outv[4] | outv[5] | outv[6] | outv[7])
                    atomicOr(&s_u[6], 1u << g);                  // 8-column groups where the block is nonzero
            }
            __syncthreads();
            if (tid == 0) {
                uint32_t m = s_u[6], j = 0;
                while (m) { wsum[j++] = __ffs(m) - 1; m &= m - 1; }
                s_u[7] = j;
            }
            __syncthreads();
            P2_LAP(15);
            if (trace && tid == 0) s_tr[7] += s_u[7];
            // rows above: R <- R - sum_k g_k * block_k, two rows per item, nonzero groups only
            const int ngm = (int)s_u[7], nrp = (r0 + 1) / 2;
            for (int it = tid; it < nrp * ngm; it += NT) {
                const int rp = it / ngm, g = (int)wsum[it % ngm];
                const int k0 = g < gv ? g * 8 : PW + (g - gv) * 8;
                const int ra = 2 * rp, rb = 2 * rp + 1;
                const bool hb = rb < r0;
                uint16_t *xa = X + bphys[ra] * LDX + k0;
                uint16_t *xb = hb ? X + bphys[rb] * LDX + k0 : xa;
                uint32_t v8[8];
                uint64_t aa[8], ab[8];
                ld8(xa, v8);
#pragma unroll
                for (int u = 0; u < 8; u++) aa[u] = v8[u];
                ld8(xb, v8);
#pragma unroll
                for (int u = 0; u < 8; u++) ab[u] = v8[u];
                for (int k = 0; k < bs; k++) {
                    const uint32_t ga = FS[ra][k], gb = hb ? FS[rb][k] : 0;
                    if (!(ga | gb)) continue;
                    const uint64_t na = ga ? p - ga : 0, nb2 = gb ? p - gb : 0;
                    ld8(X + bphys[r0 + k] * LDX + k0, v8);
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        aa[u] += na * v8[u];
                        ab[u] += nb2 * v8[u];
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; u++) v8[u] = fmod64(aa[u], F);
                st8(xa, v8);
                if (hb) {
#pragma unroll
                    for (int u = 0; u < 8; u++) v8[u] = fmod64(ab[u], F);
                    st8(xb, v8);
                }
            }
            __syncthreads();
            P2_LAP(5);
        }
        P2_LAP(5);
        if (!dense) break;                       // wide mode: every candidate was in the one chunk
    }
    // ---- 3. outputs: T (A operand tile of the Rn GEMM; wide mode wrote it), S, pivot columns, rowpiv
    for (int i = tid; dense && i < PK * PK; i += NT) {
        const int b = i / PK, s = i % PK;
        const uint16_t v = (b < (int)nb && s < (int)nb) ? X[bphys[b] * LDX + PW + bphys[s]] : 0;
        const uint32_t o = tc::toff((uint32_t)b, (uint32_t)s);
        Tlo[o] = (uint8_t)(v & 0xff);
        Thi[o] = (uint8_t)(v >> 8);
    }
    if (!published && tid < (int)nb) {
        const uint32_t rr = crow[bphys[tid]];
        const uint32_t r = src.rid ? src.rid[rr] : rr;
        cur->sel[tid] = r;
        cur->pc[tid] = (uint32_t)(c0 + bpc[tid]);
        if (!src.owner || src.owner[r] == src.me)
            rowpiv[r] = (uint32_t)(c0 + bpc[tid]);      // marks S (pivot column >= c0)
    }
    P2_LAP(6);
    if (trace && tid == 0) {
        s_tr[9] += 1; s_tr[10] += ncand_tot; s_tr[11] += nb; s_tr[12] += width; s_tr[17] += dense ? 1 : 0;
        for (int k = 0; k < 18; k++) trace[k] += s_tr[k];
    }
#undef P2_LAP
    if (!published && tid == 0) {
        cur->c0 = c0;
        cur->c1 = c0 + width;
        cur->kp = nb;
        cur->nrows = 0;
        cur->ntouch = 0;
        cur->ncand = ncand_tot;
    }
    if (epoch && !published) {
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&cur->ready), "r"(epoch) : "memory");
        }
    }
}

// F[slot] = D[i, pivot columns] for every row i not selected in this panel with
// a nonzero coefficient (limb planes of the trailing GEMM's A tiles), rows[slot] = i.
// Deferred updates (Fd != NULL): F also goes to K-block j of the row-indexed A tiles
// Fd[(i / 128) * G + j] (D row i), and kb_c0[j] = c0.
__global__ void k_gather2(int64_t mN, const uint16_t *__restrict__ D, int64_t ldD,
                          const uint32_t *__restrict__ rowpiv, P2State *__restrict__ ps,
                          uint8_t *__restrict__ Flo, uint8_t *__restrict__ Fhi, uint32_t *__restrict__ rows,
                          const uint8_t *__restrict__ owner, int me, uint8_t *__restrict__ Fdlo = nullptr,
                          uint8_t *__restrict__ Fdhi = nullptr, int G = 1, int j = 0, int64_t *__restrict__ kb_c0 = nullptr,
                          int ref = 0, uint32_t epoch = 0, const uint32_t *__restrict__ spos = nullptr,
                          const uint32_t *__restrict__ skey = nullptr, const uint32_t *__restrict__ irow = nullptr,
                          const uint32_t *__restrict__ ikey = nullptr)
{
    tc::pdl_trigger();
    tc::pdl_wait();
    if (epoch) {                                  // the panel publishes S and its pivots before its T solve
        if (threadIdx.x == 0) {
            for (uint32_t it = 0;; it++) {
                uint32_t v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&ps->ready) : "memory");
                if (v == epoch) break;
                if (it > (1u << 24)) { dev_err_latch(DEVERR_GATHER_WAIT); break; }   // bounded: never hang
                __nanosleep(128);
            }
        }
        __syncthreads();
    }
    constexpr int CPL = PK / 32;
    const int lane = threadIdx.x & 31;
    const uint32_t kp = ps->kp;
    if (kb_c0 && blockIdx.x == 0 && threadIdx.x == 0) kb_c0[j] = ps->c0;
    // prefix mode (skey != NULL: D's rows sorted by their initial leading column, skey the sorted
    // leads): the rows that can have a nonzero coefficient are exactly [0, #{ilead < c1}), and row i
    // takes slot i -- the trailing GEMM's 128-row tiles are consecutive rows of D (untouched rows
    // and this panel's pivot rows get zero factors and the row index NONE: no D traffic)
    int64_t nlim = mN;
    if (skey) {
        __shared__ uint32_t s_nt;
        if (threadIdx.x == 0) {
            const int64_t c = ps->c1;
            int64_t lo = 0, hi = mN;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)skey[mid] < c) lo = mid + 1;
                else hi = mid;
            }
            s_nt = kp ? (uint32_t)lo : 0u;
            if (blockIdx.x == 0) ps->nrows = s_nt;
        }
        __syncthreads();
        nlim = s_nt;
    }
    // row echelon form with rows indexed by their initial lead (irow / ikey, D in place, row slots
    // by atomics): only the rows with ikey < c1 can have a nonzero coefficient at this panel's pivots
    if (irow) {
        __shared__ uint32_t s_ni;
        if (threadIdx.x == 0) {
            const int64_t c = ps->c1;
            int64_t lo = 0, hi = mN;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)ikey[mid] < c) lo = mid + 1;
                else hi = mid;
            }
            s_ni = (uint32_t)lo;
        }
        __syncthreads();
        nlim = s_ni;
    }
    if (kp == 0) return;
    uint32_t touched = 0;
    for (int64_t ii = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ii < nlim;
         ii += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = irow ? (int64_t)irow[ii] : ii;
    if (owner && owner[i] != me) continue;                     // another rank's row
    const uint32_t rp = rowpiv[i];
    const bool skip = rp != GBLA_NONE && (rp >= (uint64_t)ps->c0 || ref);   // selected now: becomes Rn;
                                                                             // REF: no back elimination
    const uint16_t *drow = D + (size_t)i * ldD;
    uint16_t v[CPL];
    bool nz = false;
#pragma unroll
    for (int u = 0; u < CPL; u++) {
        const uint32_t b = lane * CPL + u;
        v[u] = (!skip && b < kp) ? drow[ps->pc[b]] : 0;
        nz |= v[u] != 0;
    }
    const bool any = __any_sync(FULL, nz);
    if (!any && !skey) continue;
    uint32_t slot = (uint32_t)i;
    if (!skey) {
        if (lane == 0) slot = atomicAdd(&ps->nrows, 1u);
        slot = __shfl_sync(FULL, slot, 0);
    }
    if (lane == 0) rows[slot] = any ? (uint32_t)i : GBLA_NONE;
    touched += any ? 1u : 0u;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int u = 0; u < CPL; u++) {
        lo |= (uint32_t)(v[u] & 0xff) << (8 * u);
        hi |= (uint32_t)(v[u] >> 8) << (8 * u);
    }
    const size_t o = (size_t)(slot / 128) * (PK * 128) + tc::toff(slot % 128, lane * CPL);
    *reinterpret_cast<uint32_t *>(Flo + o) = lo;
    *reinterpret_cast<uint32_t *>(Fhi + o) = hi;
    if (Fdlo && any) {
        const uint32_t q = spos ? spos[i] : (uint32_t)i;       // slot of row i in the flush's row order
        const size_t od = (size_t)((q / 128) * G + j) * (PK * 128) + tc::toff(q % 128, lane * CPL);
        *reinterpret_cast<uint32_t *>(Fdlo + od) = lo;
        *reinterpret_cast<uint32_t *>(Fdhi + od) = hi;
    }
    }
    if (lane == 0 && touched) atomicAdd(&ps->ntouch, touched);
}

// Deferred updates: the factors of this panel's selected rows S_b in the earlier K-blocks
// i < nk of the super-panel, moved from the row-indexed tiles Fd into the A tile Af
// (row b, K-block i) and cleared in Fd: after the fix-up GEMM brings D[S] up to date in the
// deferred columns, S_b becomes a pivot row and the flush must not subtract them again.
// Block (b, i), 32 threads x 4 K entries.
__global__ void k_fix_gather(const P2State *__restrict__ ps, int G, uint8_t *__restrict__ Fdlo,
                             uint8_t *__restrict__ Fdhi, uint8_t *__restrict__ Aflo, uint8_t *__restrict__ Afhi,
                             const uint32_t *__restrict__ spos)
{
    const uint32_t b = blockIdx.x, i = blockIdx.y;
    if (b >= ps->kp) return;
    const uint32_t r = spos ? spos[ps->sel[b]] : ps->sel[b];
    const uint32_t k = threadIdx.x * 4;
    const size_t os = (size_t)((r / 128) * G + i) * (PK * 128) + tc::toff(r % 128, k);
    const size_t od = (size_t)i * (PK * 128) + tc::toff(b, k);
    uint32_t *sl = reinterpret_cast<uint32_t *>(Fdlo + os), *sh = reinterpret_cast<uint32_t *>(Fdhi + os);
    *reinterpret_cast<uint32_t *>(Aflo + od) = *sl;
    *reinterpret_cast<uint32_t *>(Afhi + od) = *sh;
    *sl = 0;
    *sh = 0;
}

// start of a super-panel: deferred columns from Cd = min(nN, c1 + G * PW) on
__global__ void k_sp_begin(const P2State *__restrict__ ps, int64_t nN, int G, int64_t *__restrict__ Cd)
{
    const int64_t c = (ps ? ps->c1 : 0) + (int64_t)G * PW;
    *Cd = c < nN ? c : nN;
}

// Row order of the deferred flushes: D rows sorted by their leading column at the start of the
// echelon (ilead).  A row whose leading column is >= c1 has zero coefficients at every pivot of
// the panels up to column c1, so no update before then changes it: the flush of a super-panel
// ending at column c1 only touches the slots [0, #{ilead < c1}) of this order (a staircase D_new
// with uniform leads: a third of mN x width on average instead of all of it).
// ilead[r] = first nonzero column of D row r (nN if none); one warp per row, 16 bytes per lane.
__global__ void k_row_first_nz(int64_t mN, int64_t nN, const uint16_t *__restrict__ D, int64_t ldD,
                               uint32_t *__restrict__ ilead, uint32_t *__restrict__ iota)
{
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < mN;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint16_t *row = D + (size_t)r * ldD;
        uint32_t res = (uint32_t)nN;
        for (int64_t base = 0; base < nN && res == (uint32_t)nN; base += 256) {
            const int64_t k0 = base + lane * 8;
            uint32_t first = 0xffffffffu;
            if (k0 + 8 <= nN && (ldD % 8) == 0) {
                const uint4 q = __ldcs(reinterpret_cast<const uint4 *>(row + k0));
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
                uint32_t m = 0;
#pragma unroll
                for (int j = 0; j < 4; j++) m |= ((w[j] & 0xffffu) ? 1u : 0u) << (2 * j) | ((w[j] >> 16) ? 2u : 0u) << (2 * j);
                if (m) first = (uint32_t)k0 + __ffs(m) - 1;
            } else {
                for (int u = 0; u < 8; u++)
                    if (k0 + u < nN && row[k0 + u] != 0) { first = (uint32_t)(k0 + u); break; }
            }
            const unsigned m = __ballot_sync(FULL, first != 0xffffffffu);
            if (m) res = __shfl_sync(FULL, first, __ffs(m) - 1);
        }
        if (lane == 0) { ilead[r] = res; iota[r] = (uint32_t)r; }
    }
}
__global__ void k_permute_rows(int64_t ldD, const uint16_t *__restrict__ D, const uint32_t *__restrict__ srow,
                               uint16_t *__restrict__ D2)
{
    const uint4 *src = reinterpret_cast<const uint4 *>(D + (size_t)srow[blockIdx.x] * ldD);
    uint4 *dst = reinterpret_cast<uint4 *>(D2 + (size_t)blockIdx.x * ldD);
    for (int64_t q = threadIdx.x; q < ldD / 8; q += blockDim.x) dst[q] = __ldcs(src + q);
}
__global__ void k_inv_perm(int64_t n, const uint32_t *__restrict__ srow, uint32_t *__restrict__ spos)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) spos[srow[s]] = (uint32_t)s;
}
// *cnt = #{s : skey[s] < c1} (skey sorted ascending): the rows a flush ending at column c1 touches
__global__ void k_prefix_count(int64_t n, const uint32_t *__restrict__ skey, const int64_t *__restrict__ c1,
                               uint32_t *__restrict__ cnt)
{
    tc::pdl_trigger();
    tc::pdl_wait();
    const int64_t c = *c1;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)skey[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    *cnt = (uint32_t)lo;
}

// transposed limb planes of D[S, c0:]: B operand tiles (64 columns x K = 128) of the Rn GEMM
// ops != NULL (look-ahead path, where the Rn GEMM commits D[S] itself): this panel's op counts
__global__ void k_gather_st2(int64_t nN, const uint16_t *__restrict__ D, int64_t ldD,
                             const P2State *__restrict__ ps, uint8_t *__restrict__ Blo, uint8_t *__restrict__ Bhi,
                             unsigned long long *__restrict__ ops, int part)
{
    tc::pdl_trigger();
    tc::pdl_wait();
    if (ops && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && ps->c0 < nN) {
        const unsigned long long w = (unsigned long long)(nN - ps->c0);
        ops[0] += (unsigned long long)ps->ntouch * ps->kp * w;                // trailing update
        ops[1] += (unsigned long long)ps->kp * ps->kp * w;                     // new pivot rows
        ops[2] += (unsigned long long)ps->ncand * ps->kp * (unsigned long long)(ps->c1 - ps->c0);   // panel RREF
        ops[3] += (unsigned long long)ps->ntouch * w;                         // D entries of the update
    }
    const uint32_t kp = ps->kp;
    if (kp == 0) return;
    const int64_t c0 = ps->c0;
    // part 1: the 64-column tiles of the next panel's window [c1, c1 + PW) (the Rn GEMM's
    // CT_WINDOW tiles: on the look-ahead chain); part 2: the others; 0: all
    const int64_t w0 = (ps->c1 - c0) / 64 * 64, w1 = (ps->c1 - c0 + PW + 63) / 64 * 64;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + (part == 1 ? w0 : 0);
    if (c0 + x >= nN) return;
    if ((part == 1 && x >= w1) || (part == 2 && x >= w0 && x < w1)) return;
    const uint32_t s = blockIdx.y * 16;
    if (s >= kp) {      // zero K rows beyond kp (the tile is reused panel to panel)
        const size_t o = (size_t)(x / 64) * (64 * PK) + tc::toff64((uint32_t)(x % 64), s);
        *reinterpret_cast<uint4 *>(Blo + o) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4 *>(Bhi + o) = make_uint4(0, 0, 0, 0);
        return;
    }
    uint8_t lo[16], hi[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
        const uint16_t v = (s + u < kp) ? D[(size_t)ps->sel[s + u] * ldD + c0 + x] : 0;
        lo[u] = (uint8_t)(v & 0xff);
        hi[u] = (uint8_t)(v >> 8);
    }
    const size_t o = (size_t)(x / 64) * (64 * PK) + tc::toff64((uint32_t)(x % 64), s);
    *reinterpret_cast<uint4 *>(Blo + o) = *reinterpret_cast<uint4 *>(lo);
    *reinterpret_cast<uint4 *>(Bhi + o) = *reinterpret_cast<uint4 *>(hi);
}

// D[S_b, c0 + x] = Rn[b][x]; op counts (block 0, thread 0)
// part 0: all columns; 1: the next panel's window [c1, c1 + PW); 2: the other columns (+ op counts)
__global__ void k_commit2(int64_t nN, uint16_t *__restrict__ D, int64_t ldD, const P2State *__restrict__ ps,
                          const uint16_t *__restrict__ Rn, int64_t ldR, unsigned long long *__restrict__ ops, int part,
                          const uint8_t *__restrict__ owner = nullptr, int me = 0)
{
    tc::pdl_trigger();
    tc::pdl_wait();
    const uint32_t b = blockIdx.y;
    const uint32_t kp = ps->kp;
    const int64_t c0 = ps->c0;
    if (ops && part != 1 && b == 0 && blockIdx.x == 0 && threadIdx.x == 0 && c0 < nN) {
        const unsigned long long w = (unsigned long long)(nN - c0);
        ops[0] += (unsigned long long)ps->ntouch * kp * w;                    // trailing update
        ops[1] += (unsigned long long)kp * kp * w;                             // new pivot rows
        ops[2] += (unsigned long long)ps->ncand * kp * (unsigned long long)(ps->c1 - c0);   // panel RREF
        ops[3] += (unsigned long long)ps->ntouch * w;                                      // D entries of the update
    }
    // grid-stride over (row b, 8-column group); a few hundred blocks, so the next panel's
    // CTA is not queued behind thousands of tiny ones
    const int64_t w = ps->c1 - c0;
    const int64_t width = nN - c0;
    if (width <= 0) return;
    const int64_t xlo = part == 1 ? w : 0;
    const int64_t xhi = part == 1 ? (w + PW < width ? w + PW : width) : width;
    const int64_t ng = (xhi - xlo + 7) / 8;
    const bool vec = (c0 % 8 == 0) && (ldD % 8 == 0) && (ldR % 8 == 0) && (w % 8 == 0);
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < (int64_t)kp * ng;
         it += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bb = (uint32_t)(it / ng);
        if (owner && owner[ps->sel[bb]] != me) continue;           // another rank's pivot row
        const int64_t x0 = xlo + (it % ng) * 8;
        uint16_t *dst = D + (size_t)ps->sel[bb] * ldD + c0;
        const uint16_t *src = Rn + (size_t)bb * ldR;
        if (vec && x0 + 8 <= xhi && (part != 2 || x0 + 8 <= w || x0 >= w + PW)) {
            *reinterpret_cast<uint4 *>(dst + x0) = *reinterpret_cast<const uint4 *>(src + x0);
        } else {
            for (int u = 0; u < 8; u++) {
                const int64_t x = x0 + u;
                if (x >= xhi) break;
                const bool in_win = x >= w && x < w + PW;
                if (part == 2 && in_win) continue;
                dst[x] = src[x];
            }
        }
    }
    (void)b;
}

__global__ void k_p2_init(P2State *ps)
{
    ps[0].c0 = ps[0].c1 = 0;
    ps[1].c0 = ps[1].c1 = 0;
    ps[0].kp = ps[1].kp = 0;
    ps[0].nrows = ps[1].nrows = 0;
    ps[0].ntouch = ps[1].ntouch = 0;
    ps[0].ready = ps[1].ready = 0;
}

// ---- distributed echelon (row-sharded D) ----------------------------
// owner[r] = rank of D row r: target tiles (128 rows in lead order) dealt cyclically
__global__ void k_owner(int64_t mN, const uint32_t *__restrict__ order, int G, uint8_t *__restrict__ owner)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < mN) owner[order[i]] = (uint8_t)((i / 128) % G);
}

// counts of this rank's active rows by leading column in the window (lead < wmax)
__global__ void k_hist_local(int64_t mN, int64_t nN, const uint32_t *__restrict__ lead,
                             const uint8_t *__restrict__ owner, int me, const P2State *__restrict__ prev,
                             uint32_t *__restrict__ hist)
{
    const int64_t c0 = prev->c1;
    const int64_t wmax = nN - c0 < PW ? nN - c0 : PW;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < mN; r += (int64_t)gridDim.x * blockDim.x) {
        if (owner[r] != me) continue;
        const uint32_t l = lead[r];
        if (l < (uint64_t)wmax) atomicAdd(&hist[l], 1u);
    }
}

__global__ void k_sum_u32(int64_t n, int G, const uint32_t *__restrict__ in, int64_t stride, uint32_t *__restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int g = 0; g < G; g++) s += in[(size_t)g * stride + i];
        out[i] = s;
    }
}

// the panel width from the global lead counts (the same rule as k_panel2, serially):
// w[0] = width, w[1] = dense flag, w[2] = 1 once c0 >= nN
__global__ void k_width(int64_t nN, const uint32_t *__restrict__ cnt, const P2State *__restrict__ prev,
                        uint32_t *__restrict__ w, int cap)
{
    const int64_t c0 = prev->c1;
    int64_t wmax = nN - c0;
    if (wmax > PW) wmax = PW;
    if (wmax <= 0) { w[0] = 0; w[1] = 0; w[2] = 1; return; }
    const int64_t w128 = wmax < 128 ? wmax : 128;
    uint32_t cum = 0, width = (uint32_t)w128;
    uint32_t c128 = 0;
    for (int64_t c = 0; c < w128; c++) c128 += cnt[c];
    const bool dense = c128 > (uint32_t)PK;
    if (!dense) {
        for (int64_t c = 0; c <= wmax; c++) {        // cum = #rows leading before c
            if (c >= w128 && cum <= (uint32_t)cap && (c == wmax || (c & 31) == 0)) width = (uint32_t)c;
            if (c < wmax) cum += cnt[c];
        }
    }
    w[0] = width;
    w[1] = dense;
    w[2] = 0;
}

// this rank's candidates (lead < width): lead, D row id and window values (ld = ldc)
__global__ void k_cand_pack(int64_t mN, const uint16_t *__restrict__ D, int64_t ldD, const uint32_t *__restrict__ lead,
                            const uint8_t *__restrict__ owner, int me, const P2State *__restrict__ prev,
                            const uint32_t *__restrict__ w, int64_t ldc, uint32_t *__restrict__ cnt,
                            uint32_t *__restrict__ olead, uint32_t *__restrict__ orid, uint16_t *__restrict__ oval)
{
    const int64_t c0 = prev->c1;
    const uint32_t width = w[0];
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < mN;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        if (owner[r] != me || lead[r] >= width) continue;
        uint32_t slot = 0;
        if (lane == 0) slot = atomicAdd(cnt, 1u);
        slot = __shfl_sync(FULL, slot, 0);
        if (lane == 0) { olead[slot] = lead[r]; orid[slot] = (uint32_t)r; }
        for (int64_t k = lane; k < ldc; k += 32)
            oval[(size_t)slot * ldc + k] = k < (int64_t)width ? D[(size_t)r * ldD + c0 + k] : 0;
    }
}

// pad the candidate block of one rank to `maxcnt` slots (lead NONE = not a candidate)
__global__ void k_cand_pad(uint32_t cnt, uint32_t maxcnt, uint32_t *__restrict__ olead)
{
    const uint32_t i = cnt + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < maxcnt) olead[i] = NONE16;
}

// this rank's rows of S (u32, zero elsewhere): summed over ranks they give D[S, c0:]
__global__ void k_srow_pack(int64_t nN, const uint16_t *__restrict__ D, int64_t ldD, const P2State *__restrict__ ps,
                            const uint8_t *__restrict__ owner, int me, uint32_t *__restrict__ buf, int64_t ldb)
{
    const uint32_t kp = ps->kp;
    const int64_t c0 = ps->c0;
    if (c0 >= nN) return;
    const int64_t width = nN - c0;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < (int64_t)kp * width;
         it += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(it / width);
        const int64_t x = it % width;
        const uint32_t r = ps->sel[b];
        buf[(size_t)b * ldb + x] = owner[r] == me ? D[(size_t)r * ldD + c0 + x] : 0u;
    }
}

// transposed limb planes of the summed S rows (as k_gather_st2, from the u32 buffer)
__global__ void k_gather_st32(int64_t nN, const P2State *__restrict__ ps, const uint32_t *__restrict__ buf,
                              int64_t ldb, uint8_t *__restrict__ Blo, uint8_t *__restrict__ Bhi)
{
    const uint32_t kp = ps->kp;
    if (kp == 0) return;
    const int64_t c0 = ps->c0;
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c0 + x >= nN) return;
    const uint32_t s = blockIdx.y * 16;
    uint8_t lo[16], hi[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
        const uint32_t v = (s + u < kp) ? buf[(size_t)(s + u) * ldb + x] : 0;
        lo[u] = (uint8_t)(v & 0xff);
        hi[u] = (uint8_t)(v >> 8);
    }
    const size_t o = (size_t)(x / 64) * (64 * PK) + tc::toff64((uint32_t)(x % 64), s);
    *reinterpret_cast<uint4 *>(Blo + o) = *reinterpret_cast<uint4 *>(lo);
    *reinterpret_cast<uint4 *>(Bhi + o) = *reinterpret_cast<uint4 *>(hi);
}

__global__ void k_colflag2(int64_t nN, const uint32_t *__restrict__ colrow, uint32_t *__restrict__ flag)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nN) flag[c] = colrow[c] != GBLA_NONE;
    else if (c == nN) flag[c] = 0;
}

// R assembly: pivot columns of one rank's rows -> flags; that rank's R rows -> R
__global__ void k_own_pivots(int64_t mN, const uint32_t *__restrict__ rowpiv, const uint8_t *__restrict__ owner,
                             int me, uint32_t *__restrict__ colrow)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < mN && owner[i] == me && rowpiv[i] != GBLA_NONE) colrow[rowpiv[i]] = (uint32_t)i;
}
__global__ void k_flag_list(uint32_t n, const uint32_t *__restrict__ pcs, uint32_t *__restrict__ flag)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[pcs[i]] = 1;
}
// rows of the staging block (pivot columns pcs[0..n)) into R at cidx[pc]
__global__ void k_scatter_rows(int64_t nN, uint32_t n, const uint32_t *__restrict__ pcs,
                               const uint16_t *__restrict__ stg, int64_t ldS, const uint32_t *__restrict__ cidx,
                               uint16_t *__restrict__ R, int64_t ldR, uint32_t *__restrict__ pivcol)
{
    const uint32_t j = blockIdx.y;
    if (j >= n) return;
    const uint32_t c = pcs[j], k = cidx[c];
    if (blockIdx.x == 0 && threadIdx.x == 0) pivcol[k] = c;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nN; x += (int64_t)gridDim.x * blockDim.x)
        R[(size_t)k * ldR + x] = stg[(size_t)j * ldS + x];
}
// one rank's pivot rows, in pivot-column order, into the staging block + their pivot columns
__global__ void k_gather_own(int64_t nN, const uint32_t *__restrict__ colrow, const uint32_t *__restrict__ oidx,
                             const uint16_t *__restrict__ D, int64_t ldD, uint16_t *__restrict__ stg, int64_t ldS,
                             uint32_t *__restrict__ pcs, int64_t cbase)
{
    const int64_t c = cbase + blockIdx.y;
    if (c >= nN) return;
    const uint32_t r = colrow[c];
    if (r == GBLA_NONE) return;
    const uint32_t j = oidx[c];
    if (blockIdx.x == 0 && threadIdx.x == 0 && pcs) pcs[j] = (uint32_t)c;
    if (!stg) return;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nN; x += (int64_t)gridDim.x * blockDim.x)
        stg[(size_t)j * ldS + x] = D[(size_t)r * ldD + x];
}

}  // namespace

// Echelon of D with width-adaptive panels (GBLA_DENSE_TC, default).
// Echelon of D with width-adaptive panels (GBLA_DENSE_TC, default), with a
// look-ahead of one panel: the trailing update of panel k is split into the
// next panel's window (done first) and the rest; the next panel (lead, panel
// factorization, gather of F) runs on a side stream on the one SM the
// trailing GEMM leaves free while the rest of the update runs.  Hazards: the
// side stream reads D only inside the window (updated and committed before
// it starts) and writes the other parity of F / rows / the panel state; the
// main stream waits for it before the next panel's GEMMs.
gbla_status panels_tc2(gbla_mat h, uint32_t *rowpiv, unsigned long long *dops, const uint16_t *invtab)
{
    cudaStream_t st = h->stream;
    modgemm_set_sms(h->ctx->sm_count);
    const int64_t mN = h->mN, nN = h->nN, ldD = h->ldD, ldR = h->ldD;
    const int64_t npad = (nN + 63) / 64 * 64 + 128;      // + the 64-column tiles a 128-column pair tile reads
    uint32_t *rows[2], *lead;
    uint16_t *Rn;
    uint8_t *Flo[2], *Fhi[2], *Tlo2[2], *Thi2[2], *Blo, *Bhi, *Rtlo, *Rthi;
    P2State *ps;
    for (int q = 0; q < 2; q++) {
        GBLA_TRY(dalloc_t(h, mN + 1, &rows[q]));
        GBLA_TRY(dalloc_t(h, (size_t)(mN + 128) * PK, &Flo[q]));
        GBLA_TRY(dalloc_t(h, (size_t)(mN + 128) * PK, &Fhi[q]));
    }
    GBLA_TRY(dalloc_t(h, mN + 1, &lead));
    for (int q = 0; q < 2; q++) {            // T of panel k+1 is written while the rest of panel k reads T
        GBLA_TRY(dalloc_t(h, (size_t)PK * PK, &Tlo2[q]));
        GBLA_TRY(dalloc_t(h, (size_t)PK * PK, &Thi2[q]));
    }
    const bool lookahead = getenv("GBLA_NO_LOOKAHEAD") == nullptr;
    // Deferred trailing updates (super-panels of G panels): each panel updates D eagerly only
    // left of the column Cd; the columns from Cd on take one K = G * 128 update per super-panel
    // (K11 multi-K: a quarter of the HBM passes and epilogue reductions of per-panel updates).
    const int G = lookahead ? sp_panels(mN, nN, h->ref_only) : 1;
    const size_t rd_stride = (size_t)npad * PK;          // bytes per plane per K-block
    const int64_t ntrD = (mN + 127) / 128, ntrD2 = (ntrD + 1) / 2 * 2;
    uint8_t *Fdlo = nullptr, *Fdhi = nullptr, *Aflo = nullptr, *Afhi = nullptr;
    int64_t *spc0 = nullptr, *spCd = nullptr;
    GBLA_TRY(dalloc_t(h, (size_t)npad * PK, &Blo));
    GBLA_TRY(dalloc_t(h, (size_t)npad * PK, &Bhi));
    GBLA_TRY(dalloc_t(h, rd_stride * G, &Rtlo));
    GBLA_TRY(dalloc_t(h, rd_stride * G, &Rthi));
    uint8_t *Rplo = nullptr, *Rphi = nullptr;            // 2^8 Rn mod p: the second B operand of the pair flush
    if (G > 1) {
        GBLA_TRY(dalloc_t(h, rd_stride * G, &Rplo));
        GBLA_TRY(dalloc_t(h, rd_stride * G, &Rphi));
    }
    uint32_t *srow = nullptr, *spos = nullptr, *skey = nullptr, *nflush = nullptr;
    bool sorted_rows = false;                 // D physically in lead order: per-panel rows in prefix mode
    if (G > 1) {                              // (c1-sized D: the panel chain is the critical path)
        uint32_t *ilead, *iota;
        GBLA_TRY(dalloc_t(h, mN, &ilead));
        GBLA_TRY(dalloc_t(h, mN, &iota));
        GBLA_TRY(dalloc_t(h, mN, &skey));
        GBLA_TRY(dalloc_t(h, mN, &srow));
        GBLA_TRY(dalloc_t(h, mN, &spos));
        GBLA_TRY(dalloc_t(h, 1, &nflush));
        k_row_first_nz<<<grid_for(mN * 32, 256) < 16u * h->ctx->sm_count ? grid_for(mN * 32, 256)
                                                                         : 16u * h->ctx->sm_count, 256, 0, st>>>(
            mN, nN, h->D, ldD, ilead, iota);
        note_launch();
        size_t tb = 0;
        GBLA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, ilead, skey, iota, srow, (int)mN, 0, 32, st));
        void *tmp;
        GBLA_TRY(dalloc(h, tb + 16, &tmp));
        GBLA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, ilead, skey, iota, srow, (int)mN, 0, 32, st));
        k_inv_perm<<<grid_for(mN, 256), 256, 0, st>>>(mN, srow, spos);
        note_launch(3);
        // D's rows physically in that order (row i of the echelon = row srow[i] of D_new; R does not
        // depend on the row order): every later row list of the panels is then nearly a prefix of
        // consecutive rows.  Measured on K11 alone: 128-row tiles of rows scattered over D run at
        // 1.1 POPS (K = 512) / 0.19 POPS (K = 128) against 1.67 / 0.54 for consecutive rows (TLB
        // reach).  Without the memory for a second D the rows stay in place and the flushes gather
        // them through srow.
        uint16_t *D2 = nullptr;
        if (dalloc_t(h, (size_t)mN * ldD, &D2) == GBLA_OK) {
            k_permute_rows<<<(unsigned)mN, 256, 0, st>>>(ldD, h->D, srow, D2);
            note_launch();
            dfree(h, h->D);
            h->D = D2;
            srow = nullptr;                   // identity from here on
            spos = nullptr;
            sorted_rows = !getenv("GBLA_NO_PREFIX_SLOTS");
        } else {
            cudaGetLastError();
        }
    }
    // Row echelon form (K14 route, one GPU): every panel's lead scan and F gather read only the rows
    // whose INITIAL leading column is left of the window's end / the panel's end (a row's lead only
    // moves right, and an earlier pivot row is never updated), found through the rows sorted by
    // that column (D stays in place; row slots by atomics).  On a staircase D this is a few hundred
    // active rows per panel instead of all mN (c2: 40,000 rows x 1 KB per lead scan).
    uint32_t *rrow = nullptr, *rkey = nullptr;
    // (mN >= 65,536 only: the prefix walk hands K11 the rows in initial-lead order, scattered over D,
    // where the full scan lists them in D order; measured c4 echelon -166 ms, c2 neutral, c1 +0.4 ms)
    if (G == 1 && h->ref_only && (mN >= 65536 || getenv("GBLA_REF_PREFIX")) && !getenv("GBLA_REF_FULLSCAN")) {
        uint32_t *ilead, *iota;
        GBLA_TRY(dalloc_t(h, mN, &ilead));
        GBLA_TRY(dalloc_t(h, mN, &iota));
        GBLA_TRY(dalloc_t(h, mN, &rkey));
        GBLA_TRY(dalloc_t(h, mN, &rrow));
        k_row_first_nz<<<grid_for(mN * 32, 256) < 16u * h->ctx->sm_count ? grid_for(mN * 32, 256)
                                                                         : 16u * h->ctx->sm_count, 256, 0, st>>>(
            mN, nN, h->D, ldD, ilead, iota);
        note_launch();
        size_t tb = 0;
        GBLA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, ilead, rkey, iota, rrow, (int)mN, 0, 32, st));
        void *tmp;
        GBLA_TRY(dalloc(h, tb + 16, &tmp));
        GBLA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, ilead, rkey, iota, rrow, (int)mN, 0, 32, st));
        GBLA_CUDA_TRY(cudaMemsetAsync(lead, 0xff, (mN + 1) * 4, st));   // NONE16: rows never scanned
    }
    if (G > 1) {
        // an even number of row tiles (the CTA-pair GEMM reads row tiles in pairs; the extra one is zero)
        GBLA_TRY(dalloc_t(h, (size_t)ntrD2 * G * PK * 128, &Fdlo));
        GBLA_TRY(dalloc_t(h, (size_t)ntrD2 * G * PK * 128, &Fdhi));
        GBLA_TRY(dalloc_t(h, (size_t)2 * G * PK * 128, &Aflo));
        GBLA_TRY(dalloc_t(h, (size_t)2 * G * PK * 128, &Afhi));
        GBLA_CUDA_TRY(cudaMemsetAsync(Aflo + (size_t)G * PK * 128, 0, (size_t)G * PK * 128, st));
        GBLA_CUDA_TRY(cudaMemsetAsync(Afhi + (size_t)G * PK * 128, 0, (size_t)G * PK * 128, st));
        GBLA_TRY(dalloc_t(h, (size_t)G, &spc0));
        GBLA_TRY(dalloc_t(h, 1, &spCd));
    }
    GBLA_TRY(dalloc_t(h, (size_t)PK * ldR, &Rn));
    GBLA_TRY(dalloc(h, 2 * sizeof(P2State), (void **)&ps));
    static unsigned long long attr = 0;   // devices done (dev_bit)
    if (!(attr & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_panel2, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
        attr |= dev_bit();
    }
    unsigned long long *trace = nullptr;
    if (getenv("GBLA_PANEL_TRACE")) {
        GBLA_TRY(dalloc_t(h, 20, &trace));
        GBLA_CUDA_TRY(cudaMemsetAsync(trace, 0, 20 * 8, st));
    }
    const int cap = panel_cap();
    cudaStream_t side = nullptr;
    cudaEvent_t evA = nullptr, evB = nullptr;
    int64_t *c1_host = nullptr;
    gbla_status status = GBLA_OK;
    auto fail = [&](const char *what) {
        set_error("echelon: %s: %s", what, cudaGetErrorString(cudaGetLastError()));
        status = GBLA_E_CUDA;
    };
    const int gemm_grid = lookahead ? h->ctx->sm_count - 1 : h->ctx->sm_count;   // one SM for the next panel
    // the panel factorization of panel k on stream s (prev = panel k-1's state)
    // panel k: leads of the window (all SMs), the factorization (one SM), F of the other rows (all SMs).
    // With look-ahead the middle step runs on the side stream, the two wide ones on the main stream
    // where they do not compete with the rest of the previous update.
    // lead scan: one warp per row in a single pass up to 8 blocks per SM (GBLA_LEAD_BPS overrides)
    const unsigned lbps = getenv("GBLA_LEAD_BPS") ? (unsigned)atoi(getenv("GBLA_LEAD_BPS")) : 8u;
    const unsigned rgrid = grid_for(mN * 32, 256) < lbps * h->ctx->sm_count ? grid_for(mN * 32, 256)
                                                                            : lbps * h->ctx->sm_count;
    auto p_lead = [&](cudaStream_t s, int64_t k) {
        P2State *prev = ps + ((k + 1) & 1);
        launch_pdl(k_lead2, dim3(rgrid), dim3(256), 0, s, mN, nN, (const uint16_t *)h->D, ldD,
                   (const uint32_t *)rowpiv, (const P2State *)prev, lead, (const uint8_t *)nullptr, 0,
                   (const uint32_t *)rrow, (const uint32_t *)rkey);
        note_launch();
    };
    auto p_factor = [&](cudaStream_t s, int64_t k) {
        P2State *prev = ps + ((k + 1) & 1), *cur = ps + (k & 1);
        kt_mark_on(h, KT_PANEL, s);
        PanelSrc src{h->D, ldD, mN, lead, nullptr, nullptr, nullptr, 0, 0, cap, G > 1 ? 64 : 32};
        k_panel2<<<1, NT, P2_SMEM, s>>>(nN, h->F, src, rowpiv, prev, cur, Tlo2[k & 1], Thi2[k & 1], invtab, trace,
                                        (uint32_t)(k + 1));
        kt_mark_on(h, KT_PANEL, s);
        note_launch();
    };
    auto p_gather = [&](cudaStream_t s, int64_t k) {
        P2State *cur = ps + (k & 1);
        // one warp per row, blocks in row order: the row list (and the D rows of each 128-row tile
        // of K11) comes out nearly sorted, which keeps K11's scattered row accesses TLB/DRAM friendly
        k_gather2<<<grid_for(mN * 32, 256), 256, 0, s>>>(mN, h->D, ldD, rowpiv, cur, Flo[k & 1], Fhi[k & 1],
                                                         rows[k & 1], nullptr, 0, Fdlo, Fdhi, G, (int)(k % G), spc0,
                                                         h->ref_only ? 1 : 0, (uint32_t)(k + 1), spos,
                                                         sorted_rows ? (const uint32_t *)skey : nullptr, rrow, rkey);
        note_launch();
    };
    // deferred columns [Cd, nN): super-panel start (Cd, cleared factor tiles) and the K = G * 128 flush
    auto sp_begin = [&](const P2State *last, cudaStream_t s) {
        k_sp_begin<<<1, 1, 0, s>>>(last, nN, G, spCd);
        note_launch();
        if (cudaMemsetAsync(Fdlo, 0, (size_t)ntrD2 * G * PK * 128, s) != cudaSuccess ||
            cudaMemsetAsync(Fdhi, 0, (size_t)ntrD2 * G * PK * 128, s) != cudaSuccess)
            return GBLA_E_CUDA;
        return GBLA_OK;
    };
    auto sp_flush = [&](const P2State *cur, int ctsel, cudaStream_t s) {
        kt_mark_on(h, KT_TRAIL, s);
        launch_pdl(k_prefix_count, dim3(1), dim3(1), 0, s, mN, (const uint32_t *)skey, &cur->c1, nflush);
        note_launch();
        const gbla_status r = modgemm_tc_sub_mk(s, mN, nflush, nN, h->F, Fdlo, Fdhi, G, G, Rtlo, Rthi,
                                                (int64_t)rd_stride, spc0, srow, h->D, ldD, spCd, &cur->c1, PW,
                                                ctsel, gemm_grid, Rplo, Rphi);
        kt_mark_on(h, KT_TRAIL, s);
        return r;
    };
    auto factor = [&](cudaStream_t s, int64_t k) {
        p_lead(s, k);
        p_factor(s, k);
        p_gather(s, k);
    };
    // the Rn window and the window update in one persistent launch (k_modgemm_win, column-tile
    // flags; c1: 14.4 -> 14.1 ms); single super-panel panels only (G == 1), side-stream schedule;
    // GBLA_WIN_FUSED=0: two launches
    const bool winfused = lookahead && G == 1 && !(getenv("GBLA_WIN_FUSED") && atoi(getenv("GBLA_WIN_FUSED")) == 0);
    // GBLA_EARLY_GATHER=0: the next panel's F gather waits for the whole panel (default: for its flag)
    const bool early_gather = !(getenv("GBLA_EARLY_GATHER") && atoi(getenv("GBLA_EARLY_GATHER")) == 0);
    bool btiles_ready = false;               // the B tiles of the next window were gathered early
    uint32_t *wflags = nullptr;
    if (winfused) {
        GBLA_TRY(dalloc_t(h, 64, &wflags));
        GBLA_CUDA_TRY(cudaMemsetAsync(wflags, 0, 64 * 4, st));
    }
    if (lookahead) {                      // the next panel is the critical path: high-priority side stream
        side = ctx_side_stream(h->ctx);
        evA = ctx_event(h->ctx, 0);
        evB = ctx_event(h->ctx, 1);
        if (!side || !evA || !evB) fail("stream/event creation");
    }
    if (status == GBLA_OK && !(c1_host = (int64_t *)ctx_pinned(h->ctx, 2 * sizeof(int64_t)))) fail("cudaMallocHost");
    if (status == GBLA_OK) {
        k_p2_init<<<1, 1, 0, st>>>(ps);
        note_launch();
        if (G > 1) status = sp_begin(nullptr, st);
        factor(st, 0);                                  // panel 0 on the main stream
    }
    // optional timeline (GBLA_ECH_TIMELINE=n): device times of the first n look-ahead iterations
    const int ntl = getenv("GBLA_ECH_TIMELINE") ? atoi(getenv("GBLA_ECH_TIMELINE")) : 0;
    std::vector<cudaEvent_t> tl;
    auto tmark = [&](int64_t it, cudaStream_t s) {
        if (it >= ntl) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        tl.push_back(e);
    };
    // batches of panels; the host checks the previous batch's end column (pinned
    // copy + event) while the current one runs, so the GPU never waits for the host
    int batch = 8;
    int64_t k = 0;
    cudaEvent_t bev[2] = {nullptr, nullptr};
    int64_t bk[2] = {0, 0};
    int nb_done = 0;
    bev[0] = ctx_event(h->ctx, 2);
    bev[1] = ctx_event(h->ctx, 3);
    if (status == GBLA_OK && (!bev[0] || !bev[1])) fail("event");
    while (status == GBLA_OK) {
        for (int q = 0; q < batch && status == GBLA_OK; q++, k++) {
            P2State *cur = ps + (k & 1);
            const int f = (int)(k & 1);
            const int j = (int)(k % G);                  // position in the super-panel
            uint8_t *Rtl = Rtlo + j * rd_stride, *Rth = Rthi + j * rd_stride;
            uint8_t *Rpl = Rplo ? Rplo + j * rd_stride : nullptr, *Rph = Rphi ? Rphi + j * rd_stride : nullptr;
            tmark(k, st);
            if (j > 0) {                                 // S up to date in the deferred columns
                k_fix_gather<<<dim3(PK, j), 32, 0, st>>>(cur, G, Fdlo, Fdhi, Aflo, Afhi, spos);
                note_launch();
                kt_mark(h, KT_TRAIL);
                status = modgemm_tc_sub_mk(st, PK, &cur->kp, nN, h->F, Aflo, Afhi, G, j, Rtlo, Rthi,
                                           (int64_t)rd_stride, spc0, cur->sel, h->D, ldD, spCd, nullptr, 0, 0,
                                           gemm_grid, Rplo, Rphi);
                kt_mark(h, KT_TRAIL);
                if (status != GBLA_OK) break;
            }
            // look-ahead: only the B tiles of the next window are on the chain (the rest: below); with
            // the early gather they were gathered already, right after the F gather of this panel
            if (!btiles_ready) {
                launch_pdl(k_gather_st2, dim3(lookahead ? grid_for(PW + 64, 128) : grid_for(nN, 128), PK / 16),
                           dim3(128), 0, st, nN, (const uint16_t *)h->D, ldD, (const P2State *)cur, Blo, Bhi,
                           lookahead ? dops : (unsigned long long *)nullptr, lookahead ? 1 : 0);
                note_launch();
            }
            btiles_ready = false;
            if (lookahead) tmark(k, st);
            if (winfused) {
                // Rn window + window update in one launch (k_modgemm_win): timed as the trailing family
                kt_mark(h, KT_TRAIL);
                status = modgemm_tc_win(st, nN, h->F, Tlo2[f], Thi2[f], Blo, Bhi, Rtl, Rth, Flo[f], Fhi[f], rows[f],
                                        cur->sel, &cur->nrows, &cur->kp, &cur->c0, &cur->c1, PW, h->D, ldD, wflags,
                                        (uint32_t)(k + 1), gemm_grid, Rpl, Rph);
            } else {
                kt_mark(h, KT_RN);
                // look-ahead: only the window part of Rn is on the chain to the next panel, and the Rn
                // GEMM writes D[S, c0:] = Rn itself (no commit kernel on the chain)
                status = lookahead ? modgemm_tc_store(st, nN, h->F, Tlo2[f], Thi2[f], Blo, Bhi, h->D, ldD, Rtl, Rth,
                                                      &cur->c0, &cur->kp, &cur->c1, PW, 1, cur->sel, 0, Rpl, Rph)
                                   : modgemm_tc_store(st, nN, h->F, Tlo2[f], Thi2[f], Blo, Bhi, Rn, ldR, Rtl, Rth,
                                                      &cur->c0, &cur->kp, &cur->c1, PW, 0);
                if (lookahead) kt_mark2(h, KT_RN, KT_TRAIL, st);    // closes Rn window, opens the window update
                else kt_mark(h, KT_RN);
            }
            if (lookahead) tmark(k, st);
            if (status != GBLA_OK) break;
            if (!lookahead) {
                kt_mark(h, KT_TRAIL);
                status = modgemm_tc_sub(st, mN, &cur->nrows, nN, h->F, Flo[f], Fhi[f], Rtlo, Rthi, rows[f], h->D,
                                        ldD, &cur->c0, nullptr, 0, 0, gemm_grid);
                kt_mark(h, KT_TRAIL);
                if (status != GBLA_OK) break;
                k_commit2<<<2 * h->ctx->sm_count, 256, 0, st>>>(nN, h->D, ldD, cur, Rn, ldR, dops, 0);
                note_launch();
                factor(st, k + 1);
            } else {
                // the next panel's window first, then the next panel beside the rest of the update
                // timer pair of the window update closed after the next panel's lead scan: a mark
                // between the two would cut the programmatic-dependent-launch overlap on the chain
                // (the window part of the trailing time includes k_lead2: a small overestimate)
                if (!winfused)
                    status = modgemm_tc_sub(st, mN, &cur->nrows, nN, h->F, Flo[f], Fhi[f], Rtl, Rth, rows[f], h->D,
                                            ldD, &cur->c0, &cur->c1, PW, 1, gemm_grid, spCd);
                if (status != GBLA_OK) break;
                tmark(k, st);
                const bool wflush = G > 1 && j == G - 1;
                if (wflush) kt_mark(h, KT_TRAIL);                 // (the flush has its own pair)
                if (wflush && (status = sp_flush(cur, 1, st)) != GBLA_OK) break;   // next window
                p_lead(st, k + 1);
                if (!wflush) kt_mark(h, KT_TRAIL);
                if (cudaEventRecord(evA, st) != cudaSuccess || cudaStreamWaitEvent(side, evA, 0) != cudaSuccess) {
                    fail("event");
                    break;
                }
                tmark(k, side);
                p_factor(side, k + 1);
                tmark(k, side);
                if (cudaEventRecord(evB, side) != cudaSuccess) { fail("event"); break; }
                tmark(k, st);
                launch_pdl(k_gather_st2, dim3(grid_for(nN, 128), PK / 16), dim3(128), 0, st, nN,
                           (const uint16_t *)h->D, ldD, (const P2State *)cur, Blo, Bhi,
                           (unsigned long long *)nullptr, 2);
                note_launch();
                kt_mark(h, KT_RN);
                status = modgemm_tc_store(st, nN, h->F, Tlo2[f], Thi2[f], Blo, Bhi, h->D, ldD, Rtl, Rth, &cur->c0,
                                          &cur->kp, &cur->c1, PW, 2, cur->sel, 0, Rpl, Rph);
                kt_mark2(h, KT_RN, KT_TRAIL, st);
                if (status != GBLA_OK) break;
                status = modgemm_tc_sub(st, mN, &cur->nrows, nN, h->F, Flo[f], Fhi[f], Rtl, Rth, rows[f], h->D,
                                        ldD, &cur->c0, &cur->c1, PW, 2, gemm_grid, spCd);
                kt_mark(h, KT_TRAIL);
                if (status != GBLA_OK) break;
                if (G > 1 && j == G - 1) {              // end of the super-panel: the deferred columns
                    if ((status = sp_flush(cur, 2, st)) != GBLA_OK || (status = sp_begin(cur, st)) != GBLA_OK) break;
                }
                tmark(k, st);
                if (early_gather) {
                    // the F gather waits on the panel's `ready` flag (S and pivots, published before
                    // its T solve) instead of its completion, so it overlaps the T solve; so does the
                    // gather of the next window's B tiles (D[S] there is final once the rest is done)
                    p_gather(st, k + 1);
                    if (G == 1) {
                        P2State *nxt = ps + ((k + 1) & 1);
                        launch_pdl(k_gather_st2, dim3(grid_for(PW + 64, 128), PK / 16), dim3(128), 0, st, nN,
                                   (const uint16_t *)h->D, ldD, (const P2State *)nxt, Blo, Bhi, dops, 1);
                        note_launch();
                        btiles_ready = true;
                    }
                    if (cudaStreamWaitEvent(st, evB, 0) != cudaSuccess) { fail("event"); break; }
                } else {
                    if (cudaStreamWaitEvent(st, evB, 0) != cudaSuccess) { fail("event"); break; }
                    p_gather(st, k + 1);
                }
                tmark(k, st);
            }
            if (cudaGetLastError() != cudaSuccess) { fail("launch"); break; }
        }
        if (status != GBLA_OK) break;
        P2State *last = ps + ((k - 1) & 1);
        const int slot = nb_done & 1;
        if (cudaMemcpyAsync(c1_host + slot, &last->c1, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaEventRecord(bev[slot], st) != cudaSuccess) {
            fail("event");
            break;
        }
        bk[slot] = k;                              // panels enqueued through this batch
        nb_done++;
        if (nb_done >= 2) {                        // the batch before this one: done soon if not yet
            const int ps2 = (nb_done - 2) & 1;
            if (cudaEventSynchronize(bev[ps2]) != cudaSuccess) { fail("sync"); break; }
            const int64_t c1d = c1_host[ps2];
            if (c1d >= nN) break;
            // size the next batch from the mean panel width so far (few no-op panels at the end)
            const double w = (double)c1d / (double)(bk[ps2] > 0 ? bk[ps2] : 1);
            const double need = (double)(nN - c1d) / (w > 1.0 ? w : 1.0) - (double)(k - bk[ps2]);
            batch = need < 1.0 ? 1 : (need > 16.0 ? 16 : (int)need + 1);
        } else {
            batch = 8;
        }
    }
    if (status == GBLA_OK && G > 1 && (k % G) != 0) {      // the last, partial super-panel
        P2State *last = ps + ((k - 1) & 1);
        status = sp_flush(last, 0, st);
    }
    if (status == GBLA_OK && cudaStreamSynchronize(st) != cudaSuccess) fail("sync");

    if (side) cudaStreamSynchronize(side);
    if (!tl.empty()) {
        cudaDeviceSynchronize();
        // per iteration (us from its start): side panel start, end; main rest start, end; gather end
        // per iteration (us from its start): B tiles, Rn window, window update done (main stream);
        // side panel start, end; main rest start, end; gather done
        for (size_t i = 0; i + 9 <= tl.size(); i += 9) {
            float a[9];
            for (int j = 0; j < 9; j++) cudaEventElapsedTime(&a[j], tl[i], tl[i + j]);
            fprintf(stderr, "[gbla timeline] it %zu: Btiles %.1f Rn-win %.1f upd-win %.1f | panel %.1f..%.1f (%.1f) | "
                    "rest %.1f..%.1f | gather done %.1f\n", i / 9, a[1] * 1e3, a[2] * 1e3, a[3] * 1e3, a[4] * 1e3,
                    a[5] * 1e3, (a[5] - a[4]) * 1e3, a[6] * 1e3, a[7] * 1e3, a[8] * 1e3);
        }
        for (cudaEvent_t e : tl) cudaEventDestroy(e);
    }

    if (trace && status == GBLA_OK) {   // diagnostics: mean cycles per phase over the panels that ran
        unsigned long long tr[20];
        GBLA_CUDA_TRY(cudaMemcpy(tr, trace, sizeof tr, cudaMemcpyDeviceToHost));
        const double n = tr[9] ? (double)tr[9] : 1.0;
        fprintf(stderr,
                "[gbla panel2 trace] %llu panels, mean cycles: width %.0f collect %.0f load %.0f reduce+LU %.0f "
                "heads %.0f dense-backsub %.0f output %.0f; wide: U/W init %.0f W_II %.0f T solve %.0f T tile %.0f; LU steps/panel %.2f "
                "candidates %.1f pivots %.1f width %.1f dense panels %llu\n",
                tr[9], tr[0] / n, tr[1] / n, tr[2] / n, tr[3] / n, tr[4] / n, tr[5] / n, tr[6] / n, tr[13] / n, tr[14] / n,
                tr[16] / n, tr[15] / n, tr[8] / n, tr[10] / n, tr[11] / n, tr[12] / n, tr[17]);
    }
    return status;
}

// ---- distributed echelon --------------------------------------------------------------
gbla_status dist_allreduce_u32(gbla_mat h, uint32_t *buf, size_t n);
gbla_status dist_allreduce_u64(gbla_mat h, unsigned long long *buf, size_t n);
gbla_status dist_allgather(gbla_mat h, const void *send, void *recv, size_t bytes);
gbla_status dist_bcast(gbla_mat h, void *buf, size_t bytes, int root);
template <class T>
static gbla_status exclusive_scan_u32(gbla_mat h, const T *in, T *out, int64_t count);

// Echelon of a row-sharded D: rank g owns the rows of the target tiles
// T = g, g+G, ... (owner[]); nothing but the exchanges below crosses ranks.  Per panel:
//   leads + lead counts of own rows -> C3a all-reduce of the counts -> the panel width
//   (same rule as k_panel2) -> C3b all-gather of every rank's candidate slices -> every
//   rank runs the same panel factorization on the same gathered candidates (identical
//   T, S, pivot columns) -> C4 all-reduce of the S rows (each row from its owner, zeros
//   elsewhere) -> Rn = T D[S, c0:] on every rank -> K11 on own rows -> own S rows = Rn.
// R: pivot-column lists all-gathered, then every rank's pivot rows broadcast (C6) and
// placed in pivot-column order.  `real` = NCCL; otherwise the G ranks are emulated in
// this process (one shared D whose rows are disjoint between ranks) and the exchanges
// are device copies / sums - the same kernels and the same data movement.
gbla_status panels_dist(gbla_mat h, uint32_t *rowpiv, unsigned long long *dops, const uint16_t *invtab, int G,
                        int me, bool real)
{
    cudaStream_t st = h->stream;
    modgemm_set_sms(h->ctx->sm_count);
    const int64_t mN = h->mN, nN = h->nN, ldD = h->ldD, ldR = h->ldD;
    const int64_t npad = (nN + 63) / 64 * 64 + 64;
    const int nloc = real ? 1 : G;                     // ranks handled by this process
    const int pcap = panel_cap();
    auto rank_of = [&](int j) { return real ? me : j; };
    uint8_t *owner;
    uint32_t *rows, *lead, *hbuf, *ghist, *wdev, *cnt, *buf32, *bsum;
    uint16_t *Rn;
    uint8_t *Flo, *Fhi, *Tlo, *Thi, *Blo, *Bhi, *Rtlo, *Rthi;
    P2State *ps;
    GBLA_TRY(dalloc_t(h, mN + 1, &owner));
    k_owner<<<grid_for(mN, 256), 256, 0, st>>>(mN, h->order, G, owner);
    note_launch();
    GBLA_TRY(dalloc_t(h, mN + 1, &rows));
    GBLA_TRY(dalloc_t(h, mN + 1, &lead));
    GBLA_CUDA_TRY(cudaMemsetAsync(lead, 0xff, (mN + 1) * 4, st));
    GBLA_TRY(dalloc_t(h, (size_t)nloc * PW, &hbuf));
    GBLA_TRY(dalloc_t(h, PW, &ghist));
    GBLA_TRY(dalloc_t(h, 4, &wdev));
    GBLA_TRY(dalloc_t(h, (size_t)G + 1, &cnt));
    const int64_t ldb = nN > 0 ? nN : 1;
    GBLA_TRY(dalloc_t(h, (size_t)nloc * PK * ldb, &buf32));
    bsum = buf32;
    if (!real && G > 1) GBLA_TRY(dalloc_t(h, (size_t)PK * ldb, &bsum));
    GBLA_TRY(dalloc_t(h, (size_t)(mN + 128) * PK, &Flo));
    GBLA_TRY(dalloc_t(h, (size_t)(mN + 128) * PK, &Fhi));
    GBLA_TRY(dalloc_t(h, (size_t)PK * PK, &Tlo));
    GBLA_TRY(dalloc_t(h, (size_t)PK * PK, &Thi));
    GBLA_TRY(dalloc_t(h, (size_t)npad * PK, &Blo));
    GBLA_TRY(dalloc_t(h, (size_t)npad * PK, &Bhi));
    GBLA_TRY(dalloc_t(h, (size_t)npad * PK, &Rtlo));
    GBLA_TRY(dalloc_t(h, (size_t)npad * PK, &Rthi));
    GBLA_TRY(dalloc_t(h, (size_t)PK * ldR, &Rn));
    GBLA_TRY(dalloc(h, 2 * sizeof(P2State), (void **)&ps));
    // candidate blocks: per local rank (send) and gathered (G blocks of maxcnt slots)
    const int64_t cap = mN > 0 ? mN : 1;
    uint32_t *sl, *sr, *gl, *gr;
    uint16_t *sv, *gv;
    GBLA_TRY(dalloc_t(h, (size_t)nloc * cap, &sl));
    GBLA_TRY(dalloc_t(h, (size_t)nloc * cap, &sr));
    GBLA_TRY(dalloc_t(h, (size_t)nloc * cap * PW, &sv));
    int64_t gcap = 0;
    gl = gr = nullptr;
    gv = nullptr;
    static unsigned long long attr = 0;   // devices done (dev_bit)
    if (!(attr & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_panel2, cudaFuncAttributeMaxDynamicSharedMemorySize, P2_SMEM));
        attr |= dev_bit();
    }
    uint32_t *hpin = (uint32_t *)ctx_pinned(h->ctx, (8 + (size_t)G) * 4);   // width info, candidate counts
    if (!hpin) { set_error("pinned host scratch"); return GBLA_E_CUDA; }
    gbla_status status = GBLA_OK;
    const unsigned rgrid = grid_for(mN * 32, 256) < 4u * h->ctx->sm_count ? grid_for(mN * 32, 256)
                                                                            : 4u * h->ctx->sm_count;
    k_p2_init<<<1, 1, 0, st>>>(ps);
    note_launch();
    for (int64_t k = 0; status == GBLA_OK; k++) {
        P2State *prev = ps + ((k + 1) & 1), *cur = ps + (k & 1);
        // C3a: lead counts of own rows, summed over ranks
        if (cudaMemsetAsync(hbuf, 0, (size_t)nloc * PW * 4, st) != cudaSuccess) { status = GBLA_E_CUDA; break; }
        for (int j = 0; j < nloc; j++) {
            k_lead2<<<rgrid, 256, 0, st>>>(mN, nN, h->D, ldD, rowpiv, prev, lead, owner, rank_of(j));
            k_hist_local<<<grid_for(mN, 256), 256, 0, st>>>(mN, nN, lead, owner, rank_of(j), prev,
                                                            hbuf + (size_t)j * PW);
            note_launch(2);
        }
        if (real) {
            if ((status = dist_allreduce_u32(h, hbuf, PW)) != GBLA_OK) break;
            GBLA_CUDA_TRY(cudaMemcpyAsync(ghist, hbuf, PW * 4, cudaMemcpyDeviceToDevice, st));
        } else {
            k_sum_u32<<<2, 256, 0, st>>>(PW, G, hbuf, PW, ghist);
            note_launch();
        }
        k_width<<<1, 1, 0, st>>>(nN, ghist, prev, wdev, pcap);
        GBLA_CUDA_TRY(cudaMemsetAsync(cnt, 0, (G + 1) * 4, st));
        GBLA_CUDA_TRY(cudaMemcpyAsync(hpin, wdev, 12, cudaMemcpyDeviceToHost, st));
        GBLA_CUDA_TRY(cudaStreamSynchronize(st));
        if (hpin[2]) break;                                           // c0 >= nN: done
        const int64_t width = hpin[0], ldc = (width + 31) / 32 * 32;
        // C3b: every rank's candidates (lead < width)
        for (int j = 0; j < nloc; j++) {
            k_cand_pack<<<rgrid, 256, 0, st>>>(mN, h->D, ldD, lead, owner, rank_of(j), prev, wdev, ldc, cnt + j,
                                                sl + (size_t)j * cap, sr + (size_t)j * cap, sv + (size_t)j * cap * PW);
            note_launch();
        }
        if (real) {
            GBLA_CUDA_TRY(cudaMemcpyAsync(cnt + G, cnt, 4, cudaMemcpyDeviceToDevice, st));
            if ((status = dist_allgather(h, cnt + G, cnt, 4)) != GBLA_OK) break;
        }
        GBLA_CUDA_TRY(cudaMemcpyAsync(hpin + 4, cnt, (size_t)G * 4, cudaMemcpyDeviceToHost, st));
        GBLA_CUDA_TRY(cudaStreamSynchronize(st));
        uint32_t maxcnt = 0;
        for (int g = 0; g < G; g++) maxcnt = hpin[4 + g] > maxcnt ? hpin[4 + g] : maxcnt;
        if (maxcnt == 0) maxcnt = 1;
        if ((int64_t)G * maxcnt > gcap) {
            gcap = (int64_t)G * maxcnt;
            GBLA_TRY(dalloc_t(h, (size_t)gcap, &gl));
            GBLA_TRY(dalloc_t(h, (size_t)gcap, &gr));
            GBLA_TRY(dalloc_t(h, (size_t)gcap * PW, &gv));
        }
        for (int j = 0; j < nloc; j++) {
            const uint32_t cj = hpin[4 + rank_of(j)];
            if (cj < maxcnt) k_cand_pad<<<grid_for(maxcnt - cj, 256), 256, 0, st>>>(cj, maxcnt, sl + (size_t)j * cap);
        }
        if (real) {
            if ((status = dist_allgather(h, sl, gl, (size_t)maxcnt * 4)) != GBLA_OK) break;
            if ((status = dist_allgather(h, sr, gr, (size_t)maxcnt * 4)) != GBLA_OK) break;
            if ((status = dist_allgather(h, sv, gv, (size_t)maxcnt * ldc * 2)) != GBLA_OK) break;
        } else {
            for (int g = 0; g < G; g++) {
                GBLA_CUDA_TRY(cudaMemcpyAsync(gl + (size_t)g * maxcnt, sl + (size_t)g * cap, maxcnt * 4,
                                              cudaMemcpyDeviceToDevice, st));
                GBLA_CUDA_TRY(cudaMemcpyAsync(gr + (size_t)g * maxcnt, sr + (size_t)g * cap, maxcnt * 4,
                                              cudaMemcpyDeviceToDevice, st));
                GBLA_CUDA_TRY(cudaMemcpyAsync(gv + (size_t)g * maxcnt * ldc, sv + (size_t)g * cap * PW,
                                              (size_t)maxcnt * ldc * 2, cudaMemcpyDeviceToDevice, st));
            }
        }
        // the same panel factorization on every rank
        PanelSrc src{gv, ldc, (int64_t)G * maxcnt, gl, gr, ghist, real ? owner : nullptr, me, 1, pcap, 0};
        kt_mark(h, KT_PANEL);
        k_panel2<<<1, NT, P2_SMEM, st>>>(nN, h->F, src, rowpiv, prev, cur, Tlo, Thi, invtab, nullptr, 0u);
        kt_mark(h, KT_PANEL);
        note_launch();
        // C4: the S rows from their owners
        for (int j = 0; j < nloc; j++) {
            k_srow_pack<<<2 * h->ctx->sm_count, 256, 0, st>>>(nN, h->D, ldD, cur, owner, rank_of(j),
                                                               buf32 + (size_t)j * PK * ldb, ldb);
            note_launch();
        }
        if (real) {
            if ((status = dist_allreduce_u32(h, buf32, (size_t)PK * ldb)) != GBLA_OK) break;
        } else if (G > 1) {
            k_sum_u32<<<4 * h->ctx->sm_count, 256, 0, st>>>((int64_t)PK * ldb, G, buf32, (int64_t)PK * ldb, bsum);
            note_launch();
        }
        k_gather_st32<<<dim3(grid_for(nN, 128), PK / 16), 128, 0, st>>>(nN, cur, bsum, ldb, Blo, Bhi);
        note_launch();
        kt_mark(h, KT_RN);
        if ((status = modgemm_tc_store(st, nN, h->F, Tlo, Thi, Blo, Bhi, Rn, ldR, Rtlo, Rthi, &cur->c0, &cur->kp,
                                       nullptr, 0, 0)) != GBLA_OK)
            break;
        kt_mark(h, KT_RN);
        // K11 on own rows (emulated: every rank's rows in one list), own S rows = Rn
        for (int j = 0; j < nloc; j++) {
            k_gather2<<<grid_for(mN * 32, 256), 256, 0, st>>>(mN, h->D, ldD, rowpiv, cur, Flo, Fhi, rows, owner,
                                                              rank_of(j), nullptr, nullptr, 1, 0, nullptr,
                                                              h->ref_only ? 1 : 0);
            note_launch();
        }
        kt_mark(h, KT_TRAIL);
        if ((status = modgemm_tc_sub(st, mN, &cur->nrows, nN, h->F, Flo, Fhi, Rtlo, Rthi, rows, h->D, ldD,
                                     &cur->c0, nullptr, 0, 0, 0)) != GBLA_OK)
            break;
        kt_mark(h, KT_TRAIL);
        for (int j = 0; j < nloc; j++) {
            k_commit2<<<2 * h->ctx->sm_count, 256, 0, st>>>(nN, h->D, ldD, cur, Rn, ldR, j == 0 ? dops : nullptr, 0,
                                                            owner, rank_of(j));
            note_launch();
        }
        if (cudaGetLastError() != cudaSuccess) { set_error("distributed echelon: launch failed"); status = GBLA_E_CUDA; }
    }
    if (status != GBLA_OK) return status;
    // op counts: the trailing updates were split over the ranks
    if (real) {                      // dops[1], dops[2] (Rn, panel) are identical on every rank
        GBLA_TRY(dist_allreduce_u64(h, dops, 1));
        GBLA_TRY(dist_allreduce_u64(h, dops + 3, 1));
    }
    // ---- R: pivot-column lists of every rank, then every rank's pivot rows in pivot order
    uint32_t *colrow, *oflag, *oidx, *gflag, *gidx, *pcs;
    GBLA_TRY(dalloc_t(h, nN + 1, &colrow));
    GBLA_TRY(dalloc_t(h, nN + 1, &oflag));
    GBLA_TRY(dalloc_t(h, nN + 1, &oidx));
    GBLA_TRY(dalloc_t(h, nN + 1, &gflag));
    GBLA_TRY(dalloc_t(h, nN + 1, &gidx));
    std::vector<uint32_t> counts(G, 0);
    auto own_lists = [&](int g) -> gbla_status {     // colrow / oidx / count of rank g's pivot rows
        GBLA_CUDA_TRY(cudaMemsetAsync(colrow, 0xff, (nN + 1) * 4, st));
        k_own_pivots<<<grid_for(mN, 256), 256, 0, st>>>(mN, rowpiv, owner, g, colrow);
        k_colflag2<<<grid_for(nN + 1, 256), 256, 0, st>>>(nN, colrow, oflag);
        note_launch(2);
        GBLA_TRY(exclusive_scan_u32<uint32_t>(h, oflag, oidx, nN + 1));
        return GBLA_OK;
    };
    // pass 1: counts and pivot columns of every rank (pcs: G blocks of up to maxc entries)
    uint32_t mycnt = 0;
    std::vector<uint32_t> hc(G + 1, 0);
    if (real) {
        GBLA_TRY(own_lists(me));
        GBLA_CUDA_TRY(cudaMemcpyAsync(cnt + G, oidx + nN, 4, cudaMemcpyDeviceToDevice, st));
        GBLA_TRY(dist_allgather(h, cnt + G, cnt, 4));
        GBLA_CUDA_TRY(cudaMemcpyAsync(hc.data(), cnt, (size_t)G * 4, cudaMemcpyDeviceToHost, st));
        GBLA_CUDA_TRY(cudaStreamSynchronize(st));
        for (int g = 0; g < G; g++) counts[g] = hc[g];
        mycnt = counts[me];
    } else {
        for (int g = 0; g < G; g++) {
            GBLA_TRY(own_lists(g));
            GBLA_CUDA_TRY(cudaMemcpyAsync(&hc[g], oidx + nN, 4, cudaMemcpyDeviceToHost, st));
            GBLA_CUDA_TRY(cudaStreamSynchronize(st));
            counts[g] = hc[g];
        }
    }
    uint32_t maxc = 1;
    for (int g = 0; g < G; g++) maxc = counts[g] > maxc ? counts[g] : maxc;
    GBLA_TRY(dalloc_t(h, (size_t)G * maxc, &pcs));
    const unsigned gx = grid_for(nN, 256) < 8 ? grid_for(nN, 256) : 8;
    auto own_pcs = [&](uint32_t *dst, uint16_t *stg, int64_t ldS) -> gbla_status {   // after own_lists
        for (int64_t cb = 0; cb < nN; cb += 65535) {
            const int64_t n = nN - cb < 65535 ? nN - cb : 65535;
            k_gather_own<<<dim3(stg ? gx : 1, (unsigned)n), stg ? 256 : 32, 0, st>>>(nN, colrow, oidx, h->D, ldD, stg,
                                                                                    ldS, dst, cb);
            note_launch();
        }
        GBLA_CUDA_TRY(cudaGetLastError());
        return GBLA_OK;
    };
    if (real) {
        uint32_t *mine;
        GBLA_TRY(dalloc_t(h, maxc, &mine));
        GBLA_TRY(own_pcs(mine, nullptr, 0));
        GBLA_TRY(dist_allgather(h, mine, pcs, (size_t)maxc * 4));
    } else {
        for (int g = 0; g < G; g++) {
            GBLA_TRY(own_lists(g));
            GBLA_TRY(own_pcs(pcs + (size_t)g * maxc, nullptr, 0));
        }
    }
    GBLA_CUDA_TRY(cudaMemsetAsync(gflag, 0, (nN + 1) * 4, st));
    for (int g = 0; g < G; g++)
        if (counts[g]) {
            k_flag_list<<<grid_for(counts[g], 256), 256, 0, st>>>(counts[g], pcs + (size_t)g * maxc, gflag);
            note_launch();
        }
    GBLA_TRY(exclusive_scan_u32<uint32_t>(h, gflag, gidx, nN + 1));
    uint32_t rk = 0;
    unsigned long long dv[4] = {0, 0, 0, 0};
    GBLA_CUDA_TRY(cudaMemcpyAsync(&rk, gidx + nN, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(dv, dops, 32, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->rank = rk;
    h->dense_ops = dv[0] + dv[1];
    h->kwork[KT_TRAIL] = dv[0];
    h->kwork[KT_RN] = dv[1];
    h->kwork[KT_PANEL] = dv[2];
    h->trail_elems = dv[3];
    h->ldR = ldR;
    GBLA_TRY(dalloc_t(h, (size_t)(rk > 0 ? rk : 1) * h->ldR, &h->R));
    GBLA_TRY(dalloc_t(h, rk + 1, &h->pivcol));
    // pass 2 (C6): rank g's pivot rows -> every rank -> R rows cidx[pivot column]
    uint16_t *stg;
    GBLA_TRY(dalloc_t(h, (size_t)maxc * ldR, &stg));
    for (int g = 0; g < G; g++) {
        if (!counts[g]) continue;
        if (!real || g == me) {
            GBLA_TRY(own_lists(g));
            GBLA_TRY(own_pcs(nullptr, stg, ldR));
        }
        if (real) GBLA_TRY(dist_bcast(h, stg, (size_t)counts[g] * ldR * 2, g));
        for (uint32_t j0 = 0; j0 < counts[g]; j0 += 65535) {
            const uint32_t n = counts[g] - j0 < 65535 ? counts[g] - j0 : 65535;
            k_scatter_rows<<<dim3(gx, n), 256, 0, st>>>(nN, n, pcs + (size_t)g * maxc + j0, stg + (size_t)j0 * ldR,
                                                         ldR, gidx, h->R, h->ldR, h->pivcol);
            note_launch();
        }
    }
    GBLA_CUDA_TRY(cudaGetLastError());
    (void)mycnt;
    return GBLA_OK;
}

template <class T>
static gbla_status exclusive_scan_u32(gbla_mat h, const T *in, T *out, int64_t count)
{
    size_t tmp = 0;
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)count, h->stream));
    void *t = nullptr;
    GBLA_TRY(dalloc(h, tmp + 16, &t));
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)count, h->stream));
    return GBLA_OK;
}
