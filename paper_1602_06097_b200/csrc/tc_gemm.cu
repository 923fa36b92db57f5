// tc_gemm.cu -- K11: modular GEMM over GF(p), p < 2^16, on the sm_100a
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Exactness (north star "exactness bound stated in the code"): residues
// a, b < 2^16 are split into unsigned 8-bit limbs a = 256*ah + al.  Over a
// K-block of KP = 128 terms each limb product sum is <= 128 * 255^2 =
// 8,323,200 < 2^31, so the s32 TMEM accumulators are exact (the cross term
// ah*bl + al*bh <= 2 * 8,323,200 < 2^31 too).  The epilogue forms
//   S = 65536*HH + 256*X + LL  <  2^40
// in u64 and reduces it once mod p (Barrett).  4 u8 MACs per modMAC.
//
// Operands live in HBM as PRE-TILED limb planes: an A tile is 128 rows x
// 128 K (16 KB per plane), a B tile 64 columns x 128 K (8 KB per plane), each
// already in the tcgen05 K-major SWIZZLE_NONE core-matrix layout, so one
// cp.async.bulk (TMA bulk copy, SASS UBLKCP) per plane stages it.
//
// k_modgemm_ws: persistent, one CTA per SM (128 KB of operand stages), warp
// specialized: warp 0 stages the A tile of a row tile once (double-buffered)
// and the B tiles through a 4-stage ring, warp 1 issues the 16 MMAs of a
// 128 x 64 output tile (4 K-steps x 4 limb products) into one of two TMEM
// accumulators (HH | X | LL, 3 x 64 columns each), and 16 epilogue warps
// drain the other accumulator (tcgen05.ld: warp w reads TMEM lanes
// 32*(w%4)..+31, a quarter of the columns each), reduce mod p and
// read-modify-write C (16-byte vectors per thread, the C row segment
// prefetched before the accumulator is ready).  Loads, MMAs and epilogue of
// consecutive tiles overlap.  Each CTA owns a contiguous range of output
// tiles in row-tile-major order (A reuse).  Column-tile subsets (CT_WINDOW /
// CT_REST) split one update into the echelon look-ahead's two parts.
//   MODE_SUB    C[rowidx[i], x] = C - S   mod p     (trailing update)
//   MODE_STORE  O[i, x] = S mod p, plus O's limb planes as B tiles
//               (the B operand of a following MODE_SUB GEMM)
#include <stdlib.h>

#include "internal.cuh"
#include "tc.cuh"

GBLA_DEV_ERR_UNIT(tcgemm_dev_err)

namespace {

constexpr int BM = 128, BN = 64, KP = 128;
constexpr uint32_t A_PLANE = BM * KP;      // 16 KB
constexpr uint32_t B_PLANE = BN * KP;      // 8 KB
constexpr uint32_t A_BYTES = 2 * A_PLANE, B_BYTES = 2 * B_PLANE;
constexpr uint32_t STAGE = A_BYTES + B_BYTES;   // 48 KB
enum { MODE_SUB = 0, MODE_STORE = 1 };

using tc::toff64;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}


// Column-tile subsets (look-ahead of the echelon): with W0 = (*win_dev - c0) / BN and
// W1 = ceil((*win_dev - c0 + win_w) / BN): CT_WINDOW = tiles [W0, W1), CT_REST = the others.
enum { CT_ALL = 0, CT_WINDOW = 1, CT_REST = 2 };

struct MMArgs {
    int64_t nrows;                    // rows (if nrows_dev is NULL)
    const uint32_t *nrows_dev;
    int64_t cols;                     // columns (total; minus *c0_dev if given)
    Field F;
    const uint8_t *Alo, *Ahi, *Blo, *Bhi;
    const uint32_t *rowidx;
    uint16_t *C;
    int64_t ldc;
    uint8_t *Tlo, *Thi;               // MODE_STORE: limb planes of the result as B tiles
    const int64_t *c0_dev;
    const uint32_t *skip_dev;
    const int64_t *win_dev;
    int64_t win_w;
    int ctsel;
    // multi-K (MK kernels): K = nkb blocks of KP.  A tile (rt, i) at (rt * a_rt_stride + i) * A_PLANE;
    // B tile of K-block i for output column tile ct at b_kb_stride * i + (ct + (c0 - kb_c0[i]) / BN) * B_PLANE
    // (each K-block's B tiles are laid out from its own column origin kb_c0[i])
    int nkb;
    int64_t a_rt_stride;
    int64_t b_kb_stride;
    const int64_t *kb_c0;
    const int64_t *cend_dev;          // optional end column (min(cols, *cend_dev))
    int exp;                          // microbenchmark experiments (0 = normal)
    // the multi-K CTA-pair kernel's second B operand: limb planes of B' = 2^8 B mod p (same tile
    // layout as Blo / Bhi); MODE_STORE writes them for its result when Tlo2 != NULL
    const uint8_t *B2lo, *B2hi;
    uint8_t *Tlo2, *Thi2;
};

constexpr int NSB = 4;                               // B stages
// epilogue warps: 8 (2 per TMEM lane quarter, 32 columns each) or 16 (4 per quarter, 16 columns)
constexpr int ws_threads(int epiw) { return 64 + 32 * epiw; }   // producer, MMA, epilogue warps
constexpr int WS_SMEM = 2 * A_BYTES + NSB * B_BYTES; // 64 KB + 64 KB (> 114 KB: one CTA per SM)
constexpr int MK_MAX = 4;                            // K-blocks of a multi-K GEMM (K <= 512)
constexpr int ws_smem(bool mk) { return mk ? MK_MAX * A_BYTES + NSB * B_BYTES : WS_SMEM; }   // 192 KB / 128 KB

// Warp-specialized persistent K11: warp 0 stages operands (A tile once per row
// tile, double-buffered; B tiles through a 4-stage ring), warp 1 issues the
// MMAs into one of two TMEM accumulators (HH | X | LL, 192 columns each), warps
// 2.. drain the other accumulator (warp w reads TMEM lanes 32*(w%4).., a part of
// the 64 columns each), so loads, MMAs and the epilogue of consecutive tiles
// overlap.  Each CTA owns a contiguous range of output tiles in row-tile-major
// order (A reuse).
//
// MK (multi-K, MODE_SUB only): K = nkb <= 4 blocks of 128 (exact: every limb sum <= 512 * 255^2 * 2
// < 2^31).  The A tiles of all K-blocks of a row tile stay resident (one buffer, 128 KB); the B
// tiles stream through the ring, nkb per output tile.
template <int MODE, int EPI_WARPS, bool PF2, bool MK = false>
__global__ void __launch_bounds__(ws_threads(EPI_WARPS), 1) k_modgemm_ws(MMArgs g)
{
    constexpr int EPI_COLS = BN / (EPI_WARPS / 4);
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t afull[2], aempty[2], bfull[NSB], bempty[NSB], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;
    tc::pdl_trigger();
    tc::pdl_wait();
    if (g.skip_dev && *g.skip_dev == 0) return;
    int64_t cols = g.cols, c0 = 0;
    if (g.cend_dev && *g.cend_dev < cols) cols = *g.cend_dev;
    uint16_t *C = g.C;
    if (g.c0_dev) {
        c0 = *g.c0_dev;
        cols -= c0;
        if (MODE == MODE_SUB || g.rowidx) C += c0;
    }
    // MODE_STORE with rowidx: row slot of the result goes straight to C[rowidx[slot], c0 + x] for
    // slot < *skip_dev (the echelon's commit D[S, c0:] = Rn fused into the Rn GEMM)
    const int64_t nwr = (MODE == MODE_STORE && g.rowidx) ? (int64_t)*g.skip_dev : INT64_MAX;
    if (cols <= 0) return;
    const int64_t nr = g.nrows_dev ? (int64_t)*g.nrows_dev : g.nrows;
    const int64_t ntr = (nr + BM - 1) / BM, ntc_all = (cols + BN - 1) / BN;
    int64_t w0 = 0, w1 = 0;
    if (g.ctsel != CT_ALL) {
        const int64_t rel = *g.win_dev - c0;           // < 0: the window starts left of this GEMM
        w0 = rel > 0 ? rel / BN : 0;
        w1 = rel + g.win_w > 0 ? (rel + g.win_w + BN - 1) / BN : 0;
        if (w0 > ntc_all) w0 = ntc_all;
        if (w1 > ntc_all) w1 = ntc_all;
        if (w1 < w0) w1 = w0;
    }
    const int64_t ntc = g.ctsel == CT_ALL ? ntc_all : g.ctsel == CT_WINDOW ? w1 - w0 : ntc_all - (w1 - w0);
    const int64_t ntiles = ntr * ntc;
    const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * per;
    const int64_t t_end = t_begin + per < ntiles ? t_begin + per : ntiles;
    if (t_begin >= t_end) return;
    auto ct_of = [&](int64_t j) -> int64_t {
        if (g.ctsel == CT_WINDOW) return w0 + j;
        if (g.ctsel == CT_REST) return j < w0 ? j : j + (w1 - w0);
        return j;
    };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&afull[i], 1);
            tc::mbar_init(&aempty[i], 1);
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], EPI_WARPS);
        }
        for (int i = 0; i < NSB; i++) {
            tc::mbar_init(&bfull[i], 1);
            tc::mbar_init(&bempty[i], 1);
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_base;
    uint8_t *Abuf = smem, *Bbuf = smem + (MK ? MK_MAX : 2) * A_BYTES;

    if (warp == 0) {
        if (MK && lane == 0) {                 // ---- producer (multi-K)
            int64_t cur_rt = -1;
            uint32_t aph = 1, bph[NSB] = {1, 1, 1, 1};
            int s = 0;
            const int nkb = g.nkb;
            int64_t boff[MK_MAX];
            for (int i = 0; i < MK_MAX; i++) {
                boff[i] = 0;
                if (i < nkb && g.kb_c0) {
                    const int64_t d = (c0 - g.kb_c0[i]) / BN;   // < 0 only for an empty K-block (zero A)
                    boff[i] = d > 0 ? d : 0;
                }
            }
            for (int64_t tile = t_begin; tile < t_end; tile++) {
                const int64_t rt = tile / ntc, ct = ct_of(tile % ntc);
                if (rt != cur_rt) {
                    tc::mbar_wait(&aempty[0], aph);
                    aph ^= 1;
                    tc::mbar_expect_tx(&afull[0], nkb * A_BYTES);
                    for (int i = 0; i < nkb; i++) {
                        const int64_t at = rt * g.a_rt_stride + i;
                        tc::bulk_g2s(Abuf + i * A_BYTES, g.Ahi + at * A_PLANE, A_PLANE, &afull[0]);
                        tc::bulk_g2s(Abuf + i * A_BYTES + A_PLANE, g.Alo + at * A_PLANE, A_PLANE, &afull[0]);
                    }
                    cur_rt = rt;
                }
                for (int i = 0; i < nkb; i++) {
                    tc::mbar_wait(&bempty[s], bph[s]);
                    bph[s] ^= 1;
                    uint8_t *bb = Bbuf + s * B_BYTES;
                    const int64_t bo = g.b_kb_stride * i + (ct + boff[i]) * B_PLANE;
                    tc::mbar_expect_tx(&bfull[s], B_BYTES);
                    tc::bulk_g2s(bb, g.Bhi + bo, B_PLANE, &bfull[s]);
                    tc::bulk_g2s(bb + B_PLANE, g.Blo + bo, B_PLANE, &bfull[s]);
                    s = (s + 1) % NSB;
                }
            }
        } else if (!MK && lane == 0) {         // ---- producer
            int64_t cur_rt = -1;
            int aslot = 1;
            uint32_t aph[2] = {1, 1}, bph[NSB] = {1, 1, 1, 1};
            int s = 0;
            for (int64_t tile = t_begin; tile < t_end; tile++) {
                const int64_t rt = tile / ntc, ct = ct_of(tile % ntc);
                if (rt != cur_rt) {
                    aslot ^= 1;
                    tc::mbar_wait(&aempty[aslot], aph[aslot]);
                    aph[aslot] ^= 1;
                    uint8_t *ab = Abuf + aslot * A_BYTES;
                    tc::mbar_expect_tx(&afull[aslot], A_BYTES);
                    tc::bulk_g2s(ab, g.Ahi + rt * A_PLANE, A_PLANE, &afull[aslot]);
                    tc::bulk_g2s(ab + A_PLANE, g.Alo + rt * A_PLANE, A_PLANE, &afull[aslot]);
                    cur_rt = rt;
                }
                tc::mbar_wait(&bempty[s], bph[s]);
                bph[s] ^= 1;
                uint8_t *bb = Bbuf + s * B_BYTES;
                tc::mbar_expect_tx(&bfull[s], B_BYTES);
                tc::bulk_g2s(bb, g.Bhi + ct * B_PLANE, B_PLANE, &bfull[s]);
                tc::bulk_g2s(bb + B_PLANE, g.Blo + ct * B_PLANE, B_PLANE, &bfull[s]);
                s = (s + 1) % NSB;
            }
        }
    } else if (warp == 1) {
        if (MK && lane == 0) {                 // ---- MMA issuer (multi-K)
            int64_t cur_rt = -1;
            uint32_t aph = 0, bph[NSB] = {0, 0, 0, 0}, tph[2] = {1, 1};
            int s = 0, ab = 0;
            const int nkb = g.nkb;
            const uint32_t idesc = tc::idesc_u8(BM, BN);
            for (int64_t tile = t_begin; tile < t_end; tile++) {
                const int64_t rt = tile / ntc;
                if (rt != cur_rt) {
                    if (cur_rt >= 0) tc::commit(&aempty[0]);   // A free once the old row tile's MMAs finish
                    tc::mbar_wait(&afull[0], aph);
                    aph ^= 1;
                    cur_rt = rt;
                }
                tc::mbar_wait(&tempty[ab], tph[ab]);
                tph[ab] ^= 1;
                const uint32_t d = tbase + ab * 3 * BN;
                for (int i = 0; i < nkb; i++) {
                    tc::mbar_wait(&bfull[s], bph[s]);
                    bph[s] ^= 1;
                    tc::fence_after();
                    const uint32_t aH = tc::smem_u32(Abuf + i * A_BYTES), aL = aH + A_PLANE;
                    const uint32_t bH = tc::smem_u32(Bbuf + s * B_BYTES), bL = bH + B_PLANE;
#pragma unroll
                    for (int k = 0; k < KP / 32; k++) {
                        const uint32_t ao = k * 2 * (BM * 16), bo = k * 2 * (BN * 16);
                        const uint64_t dAh = tc::desc_kmajor(aH + ao, BM * 16, 128);
                        const uint64_t dAl = tc::desc_kmajor(aL + ao, BM * 16, 128);
                        const uint64_t dBh = tc::desc_kmajor(bH + bo, BN * 16, 128);
                        const uint64_t dBl = tc::desc_kmajor(bL + bo, BN * 16, 128);
                        const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                        tc::mma_i8(d + 0, dAh, dBh, idesc, acc);          // HH
                        tc::mma_i8(d + BN, dAh, dBl, idesc, acc);         // X
                        tc::mma_i8(d + 2 * BN, dAl, dBl, idesc, acc);     // LL
                        tc::mma_i8(d + BN, dAl, dBh, idesc, 1);           // X (not back to back)
                    }
                    tc::commit(&bempty[s]);
                    s = (s + 1) % NSB;
                }
                tc::commit(&tfull[ab]);
                ab ^= 1;
            }
        } else if (!MK && lane == 0) {         // ---- MMA issuer
            int64_t cur_rt = -1;
            int aslot = 1;
            uint32_t aph[2] = {0, 0}, bph[NSB] = {0, 0, 0, 0}, tph[2] = {1, 1};
            int s = 0, ab = 0;
            const uint32_t idesc = tc::idesc_u8(BM, BN);
            for (int64_t tile = t_begin; tile < t_end; tile++) {
                const int64_t rt = tile / ntc;
                if (rt != cur_rt) {
                    if (cur_rt >= 0) tc::commit(&aempty[aslot]);   // old A free once its MMAs finish
                    aslot ^= 1;
                    tc::mbar_wait(&afull[aslot], aph[aslot]);
                    aph[aslot] ^= 1;
                    cur_rt = rt;
                }
                tc::mbar_wait(&bfull[s], bph[s]);
                bph[s] ^= 1;
                tc::mbar_wait(&tempty[ab], tph[ab]);              // accumulator drained
                tph[ab] ^= 1;
                tc::fence_after();
                const uint32_t aH = tc::smem_u32(Abuf + aslot * A_BYTES), aL = aH + A_PLANE;
                const uint32_t bH = tc::smem_u32(Bbuf + s * B_BYTES), bL = bH + B_PLANE;
                const uint32_t d = tbase + ab * 3 * BN;
#pragma unroll
                for (int k = 0; k < KP / 32; k++) {
                    const uint32_t ao = k * 2 * (BM * 16), bo = k * 2 * (BN * 16);
                    const uint64_t dAh = tc::desc_kmajor(aH + ao, BM * 16, 128);
                    const uint64_t dAl = tc::desc_kmajor(aL + ao, BM * 16, 128);
                    const uint64_t dBh = tc::desc_kmajor(bH + bo, BN * 16, 128);
                    const uint64_t dBl = tc::desc_kmajor(bL + bo, BN * 16, 128);
                    tc::mma_i8(d + 0, dAh, dBh, idesc, k > 0);          // HH
                    tc::mma_i8(d + BN, dAh, dBl, idesc, k > 0);         // X
                    tc::mma_i8(d + 2 * BN, dAl, dBl, idesc, k > 0);     // LL
                    tc::mma_i8(d + BN, dAl, dBh, idesc, 1);             // X (not back to back)
                }
                tc::commit(&bempty[s]);                                 // B stage free
                tc::commit(&tfull[ab]);                                 // accumulator ready
                s = (s + 1) % NSB;
                ab ^= 1;
            }
        }
    } else {                                   // ---- epilogue warps 2..9
        const int e = warp - 2, quarter = warp & 3, part = e >> 2;
        const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && (g.ldc % 8 == 0);
        uint32_t tph[2] = {0, 0};
        int ab = 0;
        // C row segments are fetched one tile ahead (two tiles of loads in flight per warp)
        uint32_t dn[EPI_COLS / 2];
        uint16_t *crow_n = nullptr;
        bool fast_n = false, live_n = false;
        int64_t x0_n = 0, slot_n = 0;
        int64_t rt_c = -1;                   // row tile whose C row this thread holds (row index cached:
        uint16_t *rowbase = nullptr;         // a CTA's tiles are row-tile-major, so rt changes rarely)
        auto fetch = [&](int64_t tile) {
            const int64_t rt = tile / ntc, ct = ct_of(tile % ntc);
            x0_n = ct * BN + part * EPI_COLS;
            slot_n = rt * BM + quarter * 32 + lane;
            live_n = slot_n < nr;
            if (rt != rt_c) {
                rt_c = rt;
                // a row index NONE (a slot of the echelon's prefix mode with zero factors): no D traffic
                const uint32_t ri = live_n && slot_n < nwr ? (g.rowidx ? g.rowidx[slot_n] : (uint32_t)slot_n) : GBLA_NONE;
                rowbase = ri != GBLA_NONE ? C + (size_t)ri * g.ldc : nullptr;
            }
            crow_n = rowbase ? rowbase + x0_n : nullptr;
            fast_n = crow_n && vec && x0_n + EPI_COLS <= cols;
#pragma unroll
            for (int w = 0; w < EPI_COLS / 2; w++) dn[w] = 0;
            if (MODE == MODE_SUB && crow_n && g.exp != 1) {
                if (fast_n) {
#pragma unroll
                    for (int u = 0; u < EPI_COLS / 8; u++) {
                        const uint4 q = reinterpret_cast<const uint4 *>(crow_n)[u];
                        dn[4 * u] = q.x; dn[4 * u + 1] = q.y; dn[4 * u + 2] = q.z; dn[4 * u + 3] = q.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < EPI_COLS; j++)
                        if (x0_n + j < cols) dn[j / 2] |= (uint32_t)crow_n[j] << (16 * (j & 1));
                }
            }
        };
        fetch(t_begin);
        for (int64_t tile = t_begin; tile < t_end; tile++) {
            uint32_t dv[EPI_COLS / 2];
#pragma unroll
            for (int w = 0; w < EPI_COLS / 2; w++) dv[w] = dn[w];
            uint16_t *crow = crow_n;
            const bool fast = fast_n, live = live_n;
            const int64_t x0 = x0_n, slot = slot_n;
            if (PF2) {
                if (tile + 1 < t_end) fetch(tile + 1);
            }
            tc::mbar_wait(&tfull[ab], tph[ab]);
            tph[ab] ^= 1;
            tc::fence_after();
            if (g.exp == 2) {                      // experiment: MMA + operand staging only
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[ab]);
                ab ^= 1;
                continue;
            }
            const uint32_t la = tbase + ((uint32_t)(quarter * 32) << 16) + ab * 3 * BN + part * EPI_COLS;
#pragma unroll
            for (int c = 0; c < EPI_COLS; c += 16) {
                uint32_t hh[16], xx[16], ll[16];
                tc::tmem_ld16(la + c, hh);
                tc::tmem_ld16(la + BN + c, xx);
                tc::tmem_ld16(la + 2 * BN + c, ll);
                tc::tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    const uint32_t s0 = fmod_limbs(hh[j], xx[j], ll[j], g.F);
                    const uint32_t s1 = fmod_limbs(hh[j + 1], xx[j + 1], ll[j + 1], g.F);
                    const int w = (c + j) / 2;
                    if (MODE == MODE_SUB) {
                        dv[w] = fsub2(dv[w], s0 | (s1 << 16), g.F.p | (g.F.p << 16));
                    } else {
                        dv[w] = s0 | (s1 << 16);
                        if (live) {
                            const uint32_t x = (uint32_t)(x0 + c + j);
                            const size_t o = (size_t)(x / BN) * B_PLANE + toff64(x % BN, (uint32_t)slot);
                            g.Tlo[o] = (uint8_t)(s0 & 0xff);
                            g.Thi[o] = (uint8_t)(s0 >> 8);
                            g.Tlo[o + 16] = (uint8_t)(s1 & 0xff);
                            g.Thi[o + 16] = (uint8_t)(s1 >> 8);
                            if (g.Tlo2) {                  // B' = 2^8 B mod p (multi-K pair kernel)
                                const uint32_t t0 = fmod32(s0 << 8, g.F), t1 = fmod32(s1 << 8, g.F);
                                g.Tlo2[o] = (uint8_t)(t0 & 0xff);
                                g.Thi2[o] = (uint8_t)(t0 >> 8);
                                g.Tlo2[o + 16] = (uint8_t)(t1 & 0xff);
                                g.Thi2[o + 16] = (uint8_t)(t1 >> 8);
                            }
                        }
                    }
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[ab]);          // accumulator may be overwritten
            ab ^= 1;
            if (g.exp == 1) {                      // experiment: no D traffic (keep the result live)
                uint32_t acc = 0;
#pragma unroll
                for (int w = 0; w < EPI_COLS / 2; w++) acc ^= dv[w];
                if (acc == 0x9e3779b9u && crow) crow[0] = 1;
            } else if (fast) {
#pragma unroll
                for (int u = 0; u < EPI_COLS / 8; u++)
                    reinterpret_cast<uint4 *>(crow)[u] = make_uint4(dv[4 * u], dv[4 * u + 1], dv[4 * u + 2], dv[4 * u + 3]);
            } else if (crow) {
#pragma unroll
                for (int j = 0; j < EPI_COLS; j++)
                    if (x0 + j < cols) crow[j] = (uint16_t)(dv[j / 2] >> (16 * (j & 1)));
            }
            if (!PF2) {
                if (tile + 1 < t_end) fetch(tile + 1);
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

// ---- K11 multi-K on a CTA pair (tcgen05 cta_group::2) -----------------------------------------
// The deferred super-panel flush C[rowidx[i], c0 + x] -= sum_{j < nkb} A_j[i] B_j[:, x] (K <= 512):
// the dominant kernel of c2-c4.  A single CTA issuing M = 128 MMAs re-reads its A operand from
// shared memory for every N = 64 column block and reaches about half of the tensor rate
// (measured 1.48 POPS without any epilogue); a CTA pair (cluster of 2 on one TPC) issues
// M = 256 MMAs (tcgen05.mma.cta_group::2): each CTA holds the A tiles of its own 128 rows
// (resident per row-tile pair, 128 KB) and HALF of every B tile (32 of the 64 columns), the
// leader's single thread issues the MMAs for both, and each CTA's TMEM receives its own
// 128 x 64 accumulators (HH | X | LL, double-buffered).  Barriers: the leader's afull / bfull
// complete when its own bulk copies landed AND the peer's forwarder (which waits on the peer's
// own barrier) arrived remotely; the MMA commits multicast to both CTAs' empty / tfull barriers;
// both CTAs' epilogue warps arrive on the leader's tempty.  Exactness as k_modgemm_ws (MK).
// Waits are bounded (~10 s, then trap: a launch failure instead of a hung GPU).
namespace pair {
__device__ __forceinline__ uint32_t cta_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t phase)
{
    const long long t0 = clock64();
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(tc::smem_u32(bar)), "r"(phase)
            : "memory");
        if (done) return;
        if (clock64() - t0 > (1ll << 34)) __trap();          // ~9 s at 1.9 GHz: never hang the GPU
    }
}
// CTA-scope wait (no L1 invalidation): for barriers whose data is this CTA's own (TMEM accumulators)
__device__ __forceinline__ void wait_cta(uint64_t *bar, uint32_t phase)
{
    const long long t0 = clock64();
    uint32_t done = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(tc::smem_u32(bar)), "r"(phase)
            : "memory");
        if (done) return;
        if (clock64() - t0 > (1ll << 34)) __trap();
    }
}
__device__ __forceinline__ void mma2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit2(uint64_t *bar)
{
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            tc::smem_u32(bar))
        : "memory");
}
}  // namespace pair

// Two accumulators instead of three (the limb products regrouped mod p): with a = 2^8 a_h + a_l and
// B' = 2^8 B mod p (precomputed per B entry, limbs b'_h, b'_l),
//   a b = 2^8 a_h b + a_l b  ==  a_h b' + a_l b  (mod p)  ==  2^8 (a_h b'_h + a_l b_h) + (a_h b'_l + a_l b_l),
// so U = sum a_h b'_h + a_l b_h and V = sum a_h b'_l + a_l b_l (4 MMAs per K step as before) and
// S == 2^8 U + V (mod p).  Exact: U, V <= 2 K 255^2 < 2^31 for K <= 16,512 (here K <= 512); the
// epilogue forms (2^8 (U mod p) + V) < 2^24 + 2^31 in 32 bits.  A pair tile is 256 rows x 128
// columns (M = 256, N = 128 MMAs: each CTA stages one whole 64-column B tile, B and B' planes), so
// 2 x 128 TMEM columns per tile: two accumulator sets (double-buffered, 512 columns).
#ifndef PR_NSB_OVERRIDE
#define PR_NSB_OVERRIDE 3
#endif
constexpr int PR_NP = 128;                                     // columns of a pair tile
constexpr int PR_NSB = PR_NSB_OVERRIDE;                      // B stages
constexpr uint32_t PR_BSTAGE = 4 * B_PLANE;                    // B_h, B_l, B'_h, B'_l of one 64-col tile
constexpr int PR_SMEM = MK_MAX * A_BYTES + PR_NSB * PR_BSTAGE; // 128 KB + 96 KB

__global__ void __launch_bounds__(ws_threads(8), 1) k_modgemm_mk2(MMArgs g)
{
    constexpr int NP = PR_NP, NSB = PR_NSB;
    constexpr int EPI_WARPS = 8, EPI_COLS = NP / (EPI_WARPS / 4);
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t afull, aempty, bfull[NSB], bempty[NSB], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;
    tc::pdl_trigger();
    tc::pdl_wait();
    const uint32_t rank = pair::cta_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // the pair's work (identical in both CTAs); an empty launch still runs the cluster handshakes
    int64_t cols = g.cols, c0 = 0;
    uint16_t *C = g.C;
    if (g.c0_dev) {
        c0 = *g.c0_dev;
        cols -= c0;
        C += c0;
    }
    const int64_t nr = g.nrows_dev ? (int64_t)*g.nrows_dev : g.nrows;
    const int64_t ntr2 = cols > 0 ? (nr + 2 * BM - 1) / (2 * BM) : 0, ntc_all = cols > 0 ? (cols + NP - 1) / NP : 0;
    int64_t w0 = 0, w1 = 0;
    if (g.ctsel != CT_ALL && cols > 0) {
        const int64_t rel = *g.win_dev - c0;
        w0 = rel > 0 ? rel / NP : 0;
        w1 = rel + g.win_w > 0 ? (rel + g.win_w + NP - 1) / NP : 0;
        if (w0 > ntc_all) w0 = ntc_all;
        if (w1 > ntc_all) w1 = ntc_all;
        if (w1 < w0) w1 = w0;
    }
    const int64_t ntc = g.ctsel == CT_ALL ? ntc_all : g.ctsel == CT_WINDOW ? w1 - w0 : ntc_all - (w1 - w0);
    const int64_t ntiles = ntr2 * ntc;
    const int64_t npairs = gridDim.x / 2, pid = blockIdx.x / 2;
    const int64_t per = (ntiles + npairs - 1) / npairs;
    const int64_t t_begin = pid * per;
    const int64_t t_end = t_begin + per < ntiles ? t_begin + per : ntiles;
    auto ct_of = [&](int64_t j) -> int64_t {
        if (g.ctsel == CT_WINDOW) return w0 + j;
        if (g.ctsel == CT_REST) return j < w0 ? j : j + (w1 - w0);
        return j;
    };
    const int nkb = g.nkb;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::smem_u32(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        const uint32_t nfill = rank == 0 ? 2 : 1;        // leader: own copies + the peer's forwarder
        tc::mbar_init(&afull, nfill);
        tc::mbar_init(&aempty, 1);
        for (int i = 0; i < NSB; i++) {
            tc::mbar_init(&bfull[i], nfill);
            tc::mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], 2 * EPI_WARPS);
        }
    }
    tc::fence_before();
    pair::cluster_sync();
    tc::fence_after();
    const uint32_t tbase = tmem_base;
    uint8_t *Abuf = smem, *Bbuf = smem + MK_MAX * A_BYTES;
    if (t_begin < t_end) {
    if (warp == 0 && lane == 0) {                    // ---- producer (both CTAs): own A rows, own B tile
        int64_t cur_rt = -1;
        uint32_t aph = 1, bph = 0;                   // bph: bit s = phase of stage s
        int s = 0;
        int64_t boff[MK_MAX];
#pragma unroll
        for (int i = 0; i < MK_MAX; i++) {
            boff[i] = 0;
            if (i < nkb && g.kb_c0) {
                const int64_t d = (c0 - g.kb_c0[i]) / BN;
                boff[i] = d > 0 ? d : 0;
            }
        }
        for (int64_t tile = t_begin; tile < t_end; tile++) {
            const int64_t rt2 = tile / ntc, ct = ct_of(tile % ntc);
            if (rt2 != cur_rt) {
                pair::wait(&aempty, aph);
                aph ^= 1;
                tc::mbar_expect_tx(&afull, nkb * A_BYTES);
                const int64_t rt = 2 * rt2 + rank;
                for (int i = 0; i < nkb; i++) {
                    const int64_t at = rt * g.a_rt_stride + i;
                    tc::bulk_g2s(Abuf + i * A_BYTES, g.Ahi + at * A_PLANE, A_PLANE, &afull);
                    tc::bulk_g2s(Abuf + i * A_BYTES + A_PLANE, g.Alo + at * A_PLANE, A_PLANE, &afull);
                }
                cur_rt = rt2;
            }
#pragma unroll 1
            for (int i = 0; i < nkb && g.exp != 3; i++) {
                pair::wait(&bempty[s], ((bph >> s) & 1) ^ 1);
                uint8_t *bb = Bbuf + s * PR_BSTAGE;
                tc::mbar_expect_tx(&bfull[s], PR_BSTAGE);
                // this CTA's 64 columns: the 64-column B tile 2 ct + rank (planes B_h, B_l, B'_h, B'_l)
                const int64_t bo = g.b_kb_stride * i + (2 * ct + rank + boff[i]) * B_PLANE;
                tc::bulk_g2s(bb, g.Bhi + bo, B_PLANE, &bfull[s]);
                tc::bulk_g2s(bb + B_PLANE, g.Blo + bo, B_PLANE, &bfull[s]);
                tc::bulk_g2s(bb + 2 * B_PLANE, g.B2hi + bo, B_PLANE, &bfull[s]);
                tc::bulk_g2s(bb + 3 * B_PLANE, g.B2lo + bo, B_PLANE, &bfull[s]);
                bph ^= 1u << s;
                s = (s + 1) % NSB;
            }
        }
    } else if (warp == 1 && lane == 0 && rank == 1) {   // ---- peer: forward own fills to the leader
        int64_t cur_rt = -1;
        uint32_t aph = 0, bph = 0;
        int s = 0;
        const uint32_t ra = pair::mapa(&afull, 0);
        for (int64_t tile = t_begin; tile < t_end; tile++) {
            const int64_t rt2 = tile / ntc;
            if (rt2 != cur_rt) {
                pair::wait(&afull, aph);
                aph ^= 1;
                pair::arrive_remote(ra);
                cur_rt = rt2;
            }
#pragma unroll 1
            for (int i = 0; i < nkb && g.exp != 3; i++) {
                pair::wait(&bfull[s], (bph >> s) & 1);
                bph ^= 1u << s;
                pair::arrive_remote(pair::mapa(&bfull[s], 0));
                s = (s + 1) % NSB;
            }
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {   // ---- MMA issuer (leader)
        int64_t cur_rt = -1;
        uint32_t aph = 0, bph = 0, tph[2] = {1, 1};
        int s = 0, ab = 0;
        const uint32_t idesc = tc::idesc_u8(2 * BM, NP);
        for (int64_t tile = t_begin; tile < t_end; tile++) {
            const int64_t rt2 = tile / ntc;
            if (rt2 != cur_rt) {
                if (cur_rt >= 0) pair::commit2(&aempty);
                pair::wait(&afull, aph);
                aph ^= 1;
                cur_rt = rt2;
            }
            pair::wait(&tempty[ab], tph[ab]);
            tph[ab] ^= 1;
            const uint32_t dU = tbase + ab * 2 * NP, dV = dU + NP;
#pragma unroll 1
            for (int i = 0; i < nkb; i++) {
                if (g.exp != 3) {                        // experiment 3: tensor rate alone (no B traffic)
                    pair::wait(&bfull[s], (bph >> s) & 1);
                    bph ^= 1u << s;
                }
                tc::fence_after();
                const uint32_t aH = tc::smem_u32(Abuf + i * A_BYTES), aL = aH + A_PLANE;
                const uint32_t bH = tc::smem_u32(Bbuf + s * PR_BSTAGE), bL = bH + B_PLANE;
                const uint32_t b2H = bH + 2 * B_PLANE, b2L = bH + 3 * B_PLANE;
#pragma unroll
                for (int k = 0; k < KP / 32; k++) {
                    const uint32_t ao = k * 2 * (BM * 16), bo = k * 2 * (BN * 16);
                    const uint64_t dAh = tc::desc_kmajor(aH + ao, BM * 16, 128);
                    const uint64_t dAl = tc::desc_kmajor(aL + ao, BM * 16, 128);
                    const uint64_t dBh = tc::desc_kmajor(bH + bo, BN * 16, 128);
                    const uint64_t dBl = tc::desc_kmajor(bL + bo, BN * 16, 128);
                    const uint64_t dB2h = tc::desc_kmajor(b2H + bo, BN * 16, 128);
                    const uint64_t dB2l = tc::desc_kmajor(b2L + bo, BN * 16, 128);
                    const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                    // alternate the accumulators: an MMA into the accumulator of the one just issued
                    // waits for it (measured: U, U, V, V runs at half the rate of U, V, U, V)
                    pair::mma2(dU, dAh, dB2h, idesc, acc);        // U += a_h b'_h
                    pair::mma2(dV, dAh, dB2l, idesc, acc);        // V += a_h b'_l
                    pair::mma2(dU, dAl, dBh, idesc, 1);           // U += a_l b_h
                    pair::mma2(dV, dAl, dBl, idesc, 1);           // V += a_l b_l
                }
                if (g.exp != 3) pair::commit2(&bempty[s]);
                s = (s + 1) % NSB;
            }
            pair::commit2(&tfull[ab]);
            ab ^= 1;
        }
    } else if (warp >= 2) {                          // ---- epilogue warps 2..9 (both CTAs)
        const int e = warp - 2, quarter = warp & 3, part = e >> 2;
        // 32-byte vectors (LDG/STG.256) when every row segment is 32-byte aligned
        const bool vec = ((reinterpret_cast<uintptr_t>(C) & 31) == 0) && (g.ldc % 16 == 0);
        const uint32_t tempty_leader[2] = {pair::mapa(&tempty[0], 0), pair::mapa(&tempty[1], 0)};
        uint32_t tph[2] = {0, 0};
        int ab = 0;
        uint32_t dn[EPI_COLS / 2];
        uint16_t *crow_n = nullptr;
        bool fast_n = false, live_n = false;
        int64_t x0_n = 0;
        int64_t rt_c = -1;
        uint16_t *rowbase = nullptr;
        auto fetch = [&](int64_t tile) {
            const int64_t rt2 = tile / ntc, ct = ct_of(tile % ntc);
            x0_n = ct * NP + part * EPI_COLS;
            const int64_t slot = (2 * rt2 + rank) * BM + quarter * 32 + lane;
            live_n = slot < nr;
            if (rt2 != rt_c) {
                rt_c = rt2;
                const uint32_t ri = live_n ? (g.rowidx ? g.rowidx[slot] : (uint32_t)slot) : GBLA_NONE;
                rowbase = ri != GBLA_NONE ? C + (size_t)ri * g.ldc : nullptr;
            }
            crow_n = rowbase ? rowbase + x0_n : nullptr;
            fast_n = crow_n && vec && x0_n + EPI_COLS <= cols;
#pragma unroll
            for (int w = 0; w < EPI_COLS / 2; w++) dn[w] = 0;
            if (crow_n && g.exp != 1) {
                if (fast_n) {
#pragma unroll
                    for (int u = 0; u < EPI_COLS / 16; u++)
                        asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                     : "=r"(dn[8 * u]), "=r"(dn[8 * u + 1]), "=r"(dn[8 * u + 2]), "=r"(dn[8 * u + 3]),
                                       "=r"(dn[8 * u + 4]), "=r"(dn[8 * u + 5]), "=r"(dn[8 * u + 6]), "=r"(dn[8 * u + 7])
                                     : "l"(crow_n + 16 * u));
                } else {
#pragma unroll
                    for (int j = 0; j < EPI_COLS; j++)
                        if (x0_n + j < cols) dn[j / 2] |= (uint32_t)crow_n[j] << (16 * (j & 1));
                }
            }
        };
        fetch(t_begin);
        const uint32_t p2 = g.F.p | (g.F.p << 16);
        for (int64_t tile = t_begin; tile < t_end; tile++) {
            uint32_t dv[EPI_COLS / 2];
#pragma unroll
            for (int w = 0; w < EPI_COLS / 2; w++) dv[w] = dn[w];
            uint16_t *crow = crow_n;
            const bool fast = fast_n;
            const int64_t x0 = x0_n;
            if (tile + 1 < t_end) fetch(tile + 1);
            pair::wait_cta(&tfull[ab], tph[ab]);
            tph[ab] ^= 1;
            tc::fence_after();
            if (g.exp != 2) {
                const uint32_t la = tbase + ((uint32_t)(quarter * 32) << 16) + ab * 2 * NP + part * EPI_COLS;
#pragma unroll
                for (int c = 0; c < EPI_COLS; c += 16) {
                    uint32_t uu[16], vv[16];
                    tc::tmem_ld16(la + c, uu);
                    tc::tmem_ld16(la + NP + c, vv);
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        const uint32_t s0 = fmod32((fmod32(uu[j], g.F) << 8) + vv[j], g.F);
                        const uint32_t s1 = fmod32((fmod32(uu[j + 1], g.F) << 8) + vv[j + 1], g.F);
                        const int w = (c + j) / 2;
                        dv[w] = fsub2(dv[w], s0 | (s1 << 16), p2);
                    }
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) mbar_arrive(&tempty[ab]);
                else pair::arrive_remote(tempty_leader[ab]);
            }
            ab ^= 1;
            if (g.exp >= 1) {
                uint32_t acc = 0;
#pragma unroll
                for (int w = 0; w < EPI_COLS / 2; w++) acc ^= dv[w];
                if (acc == 0x9e3779b9u && crow) crow[0] = 1;
            } else if (fast) {
#pragma unroll
                for (int u = 0; u < EPI_COLS / 16; u++)
                    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(crow + 16 * u), "r"(dv[8 * u]),
                                 "r"(dv[8 * u + 1]), "r"(dv[8 * u + 2]), "r"(dv[8 * u + 3]), "r"(dv[8 * u + 4]),
                                 "r"(dv[8 * u + 5]), "r"(dv[8 * u + 6]), "r"(dv[8 * u + 7])
                                 : "memory");
            } else if (crow) {
#pragma unroll
                for (int j = 0; j < EPI_COLS; j++)
                    if (x0 + j < cols) crow[j] = (uint16_t)(dv[j / 2] >> (16 * (j & 1)));
            }
        }
    }
    }
    tc::fence_before();
    pair::cluster_sync();                            // the MMAs read both CTAs' shared memory
    if (warp == 0) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
    }
}

// ---- the echelon's window step in ONE launch (look-ahead path, GBLA_WIN_FUSED) ---------------
// Tiles q = 0 .. nW-1: Rn window column tile ct = w0 + q (MODE_STORE: A = T, B = the gathered B
// tiles of D[S, c0:]; writes D[S, c0:] = Rn and the Rn limb tiles, then publishes flag[q] = epoch);
// tiles q >= nW: the window update D[rows, c0:] -= F Rn for row tile (q - nW) / nW and column tile
// w0 + (q - nW) % nW (MODE_SUB), whose B operand (the Rn tile) is waited for by its flag.  CTA b
// takes tiles b, b + grid, ...: a CTA's first tile is its only Rn tile, so every wait is on a tile
// another CTA reaches first; all CTAs are co-resident (one per SM, grid <= SMs), so no cycle.
struct WinArgs {
    Field F;
    const uint8_t *Tlo, *Thi;              // A operand of the Rn tiles (one 128 x 128 tile)
    const uint8_t *Bglo, *Bghi;            // gathered B tiles of D[S, c0:] (column tiles from c0)
    uint8_t *Rlo, *Rhi;                    // Rn limb tiles (written here, B operand of the update)
    uint8_t *Rlo2, *Rhi2;                  // optional: limb tiles of 2^8 Rn mod p (multi-K pair kernel)
    const uint8_t *Flo, *Fhi;              // A operand of the update (row tiles of the F list)
    const uint32_t *rows;                  // D rows of the update (slot -> row)
    const uint32_t *sel;                   // D rows of the pivot rows (slot -> row)
    const uint32_t *nrows_dev, *kp_dev;
    const int64_t *c0_dev, *win_dev;
    int64_t win_w, cols;
    uint16_t *D;
    int64_t ldD;
    uint32_t *flags;
    uint32_t epoch;
};

__device__ __forceinline__ uint32_t ld_acq(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(ws_threads(8), 1) k_modgemm_win(WinArgs g)
{
    constexpr int EPI_WARPS = 8, EPI_COLS = BN / (EPI_WARPS / 4);
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t afull[2], aempty[2], bfull[NSB], bempty[NSB], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;
    tc::pdl_trigger();
    tc::pdl_wait();
    do {                                       // the window step (skipped as a whole if empty)
    const uint32_t kp = *g.kp_dev;
    if (kp == 0) break;
    const int64_t c0 = *g.c0_dev;
    const int64_t cols = g.cols - c0;
    if (cols <= 0) break;
    uint16_t *C = g.D + c0;
    const int64_t nr = (int64_t)*g.nrows_dev;
    const int64_t ntr = (nr + BM - 1) / BM, ntc_all = (cols + BN - 1) / BN;
    const int64_t rel = *g.win_dev - c0;
    int64_t w0 = rel > 0 ? rel / BN : 0, w1 = rel + g.win_w > 0 ? (rel + g.win_w + BN - 1) / BN : 0;
    if (w0 > ntc_all) w0 = ntc_all;
    if (w1 > ntc_all) w1 = ntc_all;
    if (w1 < w0) w1 = w0;
    const int64_t nW = w1 - w0;
    if (nW == 0) break;
    const int64_t ntiles = nW + ntr * nW;
    const int64_t cnt = (int64_t)blockIdx.x < ntiles ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
    if (cnt == 0) break;
    auto tile_q = [&](int64_t i) -> int64_t { return (int64_t)blockIdx.x + i * (int64_t)gridDim.x; };
    // -1: the T tile (Rn), else the row tile of the update; column tile
    auto rt_of = [&](int64_t q) -> int64_t { return q < nW ? -1 : (q - nW) / nW; };
    auto ct_of = [&](int64_t q) -> int64_t { return w0 + (q < nW ? q : (q - nW) % nW); };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) {
        for (int i = 0; i < 2; i++) {
            tc::mbar_init(&afull[i], 1);
            tc::mbar_init(&aempty[i], 1);
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], EPI_WARPS);
        }
        for (int i = 0; i < NSB; i++) {
            tc::mbar_init(&bfull[i], 1);
            tc::mbar_init(&bempty[i], 1);
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_base;
    uint8_t *Abuf = smem, *Bbuf = smem + 2 * A_BYTES;
    if (warp == 0) {
        if (lane == 0) {                       // ---- producer
            int64_t cur_rt = -2;
            int aslot = 1;
            uint32_t aph[2] = {1, 1}, bph[NSB] = {1, 1, 1, 1};
            int s = 0;
            for (int64_t i = 0; i < cnt; i++) {
                const int64_t q = tile_q(i), rt = rt_of(q), ct = ct_of(q);
                if (rt != cur_rt) {
                    aslot ^= 1;
                    tc::mbar_wait(&aempty[aslot], aph[aslot]);
                    aph[aslot] ^= 1;
                    uint8_t *ab = Abuf + aslot * A_BYTES;
                    tc::mbar_expect_tx(&afull[aslot], A_BYTES);
                    if (rt < 0) {
                        tc::bulk_g2s(ab, g.Thi, A_PLANE, &afull[aslot]);
                        tc::bulk_g2s(ab + A_PLANE, g.Tlo, A_PLANE, &afull[aslot]);
                    } else {
                        tc::bulk_g2s(ab, g.Fhi + rt * A_PLANE, A_PLANE, &afull[aslot]);
                        tc::bulk_g2s(ab + A_PLANE, g.Flo + rt * A_PLANE, A_PLANE, &afull[aslot]);
                    }
                    cur_rt = rt;
                }
                tc::mbar_wait(&bempty[s], bph[s]);
                bph[s] ^= 1;
                uint8_t *bb = Bbuf + s * B_BYTES;
                if (rt >= 0) {                 // the Rn tile: published by the CTA that computed it
                    const uint32_t *fl = g.flags + (ct - w0);
                    for (uint32_t it = 0; ld_acq(fl) != g.epoch; it++) {
                        __nanosleep(64);
                        if (it > (1u << 24)) { dev_err_latch(DEVERR_WIN_FLAG); break; }   // never hang the GPU
                    }
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                tc::mbar_expect_tx(&bfull[s], B_BYTES);
                const uint8_t *bh = rt < 0 ? g.Bghi : g.Rhi, *bl = rt < 0 ? g.Bglo : g.Rlo;
                tc::bulk_g2s(bb, bh + ct * B_PLANE, B_PLANE, &bfull[s]);
                tc::bulk_g2s(bb + B_PLANE, bl + ct * B_PLANE, B_PLANE, &bfull[s]);
                s = (s + 1) % NSB;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                       // ---- MMA issuer
            int64_t cur_rt = -2;
            int aslot = 1;
            uint32_t aph[2] = {0, 0}, bph[NSB] = {0, 0, 0, 0}, tph[2] = {1, 1};
            int s = 0, ab = 0;
            const uint32_t idesc = tc::idesc_u8(BM, BN);
            for (int64_t i = 0; i < cnt; i++) {
                const int64_t rt = rt_of(tile_q(i));
                if (rt != cur_rt) {
                    if (cur_rt != -2) tc::commit(&aempty[aslot]);
                    aslot ^= 1;
                    tc::mbar_wait(&afull[aslot], aph[aslot]);
                    aph[aslot] ^= 1;
                    cur_rt = rt;
                }
                tc::mbar_wait(&bfull[s], bph[s]);
                bph[s] ^= 1;
                tc::mbar_wait(&tempty[ab], tph[ab]);
                tph[ab] ^= 1;
                tc::fence_after();
                const uint32_t aH = tc::smem_u32(Abuf + aslot * A_BYTES), aL = aH + A_PLANE;
                const uint32_t bH = tc::smem_u32(Bbuf + s * B_BYTES), bL = bH + B_PLANE;
                const uint32_t d = tbase + ab * 3 * BN;
#pragma unroll
                for (int k = 0; k < KP / 32; k++) {
                    const uint32_t ao = k * 2 * (BM * 16), bo = k * 2 * (BN * 16);
                    const uint64_t dAh = tc::desc_kmajor(aH + ao, BM * 16, 128);
                    const uint64_t dAl = tc::desc_kmajor(aL + ao, BM * 16, 128);
                    const uint64_t dBh = tc::desc_kmajor(bH + bo, BN * 16, 128);
                    const uint64_t dBl = tc::desc_kmajor(bL + bo, BN * 16, 128);
                    tc::mma_i8(d + 0, dAh, dBh, idesc, k > 0);
                    tc::mma_i8(d + BN, dAh, dBl, idesc, k > 0);
                    tc::mma_i8(d + 2 * BN, dAl, dBl, idesc, k > 0);
                    tc::mma_i8(d + BN, dAl, dBh, idesc, 1);
                }
                tc::commit(&bempty[s]);
                tc::commit(&tfull[ab]);
                s = (s + 1) % NSB;
                ab ^= 1;
            }
        }
    } else {                                   // ---- epilogue warps 2..9
        const int e = warp - 2, quarter = warp & 3, part = e >> 2;
        uint32_t tph[2] = {0, 0};
        int ab = 0;
        for (int64_t i = 0; i < cnt; i++) {
            const int64_t q = tile_q(i), rt = rt_of(q), ct = ct_of(q);
            const bool rn = rt < 0;
            const int64_t x0 = ct * BN + part * EPI_COLS;
            const int64_t slot = (rn ? 0 : rt * BM) + quarter * 32 + lane;
            const bool live = rn ? slot < BM : slot < nr;            // rows of the accumulator
            uint16_t *crow = nullptr;
            if (rn ? slot < (int64_t)kp : live) {
                const uint32_t ri = rn ? g.sel[slot] : g.rows[slot];
                if (ri != GBLA_NONE) crow = C + (size_t)ri * g.ldD + x0;        // NONE: zero factors
            }
            const bool fast = crow && x0 + EPI_COLS <= cols && (g.ldD % 8 == 0) &&
                              ((reinterpret_cast<uintptr_t>(crow) & 15) == 0);
            uint32_t dv[EPI_COLS / 2];
#pragma unroll
            for (int w = 0; w < EPI_COLS / 2; w++) dv[w] = 0;
            if (!rn && crow) {                 // the D row segment to update
                if (fast) {
#pragma unroll
                    for (int u = 0; u < EPI_COLS / 8; u++) {
                        const uint4 v = reinterpret_cast<const uint4 *>(crow)[u];
                        dv[4 * u] = v.x; dv[4 * u + 1] = v.y; dv[4 * u + 2] = v.z; dv[4 * u + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < EPI_COLS; j++)
                        if (x0 + j < cols) dv[j / 2] |= (uint32_t)crow[j] << (16 * (j & 1));
                }
            }
            tc::mbar_wait(&tfull[ab], tph[ab]);
            tph[ab] ^= 1;
            tc::fence_after();
            const uint32_t la = tbase + ((uint32_t)(quarter * 32) << 16) + ab * 3 * BN + part * EPI_COLS;
#pragma unroll
            for (int c = 0; c < EPI_COLS; c += 16) {
                uint32_t hh[16], xx[16], ll[16];
                tc::tmem_ld16(la + c, hh);
                tc::tmem_ld16(la + BN + c, xx);
                tc::tmem_ld16(la + 2 * BN + c, ll);
                tc::tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    const uint32_t s0 = fmod_limbs(hh[j], xx[j], ll[j], g.F);
                    const uint32_t s1 = fmod_limbs(hh[j + 1], xx[j + 1], ll[j + 1], g.F);
                    const int w = (c + j) / 2;
                    if (!rn) {
                        dv[w] = fsub2(dv[w], s0 | (s1 << 16), g.F.p | (g.F.p << 16));
                    } else {
                        dv[w] = s0 | (s1 << 16);
                        const uint32_t x = (uint32_t)(x0 + c + j);
                        const size_t o = (size_t)(x / BN) * B_PLANE + toff64(x % BN, (uint32_t)slot);
                        g.Rlo[o] = (uint8_t)(s0 & 0xff);
                        g.Rhi[o] = (uint8_t)(s0 >> 8);
                        g.Rlo[o + 16] = (uint8_t)(s1 & 0xff);
                        g.Rhi[o + 16] = (uint8_t)(s1 >> 8);
                        if (g.Rlo2) {
                            const uint32_t t0 = fmod32(s0 << 8, g.F), t1 = fmod32(s1 << 8, g.F);
                            g.Rlo2[o] = (uint8_t)(t0 & 0xff);
                            g.Rhi2[o] = (uint8_t)(t0 >> 8);
                            g.Rlo2[o + 16] = (uint8_t)(t1 & 0xff);
                            g.Rhi2[o + 16] = (uint8_t)(t1 >> 8);
                        }
                    }
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[ab]);
            ab ^= 1;
            if (fast) {
#pragma unroll
                for (int u = 0; u < EPI_COLS / 8; u++)
                    reinterpret_cast<uint4 *>(crow)[u] = make_uint4(dv[4 * u], dv[4 * u + 1], dv[4 * u + 2], dv[4 * u + 3]);
            } else if (crow) {
#pragma unroll
                for (int j = 0; j < EPI_COLS; j++)
                    if (x0 + j < cols) crow[j] = (uint16_t)(dv[j / 2] >> (16 * (j & 1)));
            }
            if (rn) {                          // publish the Rn tile: every epilogue thread's stores, then the flag
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
                if (warp == 2 && lane == 0)
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(g.flags + (ct - w0)), "r"(g.epoch) : "memory");
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tbase);
    } while (0);
}

// INT-pipe reference engine for the same op (tests / GBLA_DENSE_INT).
__global__ void k_modgemm_int(int64_t rows, int64_t cols, int64_t K, Field F, const uint16_t *__restrict__ A,
                              int64_t lda, const uint16_t *__restrict__ B, int64_t ldb,
                              const uint32_t *__restrict__ rowidx, uint16_t *__restrict__ C, int64_t ldc)
{
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = blockIdx.y;
    if (x >= cols || i >= rows) return;
    uint64_t acc = 0;
    for (int64_t k = 0; k < K; k++) acc += (uint64_t)A[i * lda + k] * B[k * ldb + x];
    const uint32_t s = fmod64(acc, F);
    uint16_t *c = C + (size_t)(rowidx ? rowidx[i] : i) * ldc + x;
    const uint32_t d = *c;
    *c = (uint16_t)(d >= s ? d - s : d + F.p - s);
}

// rows x K (lda) u16 -> A tiles (limb planes), zero padded; K-block i of row tile rt is tile
// rt * nkb + i (nkb = 1: one 128 x 128 tile per row tile)
__global__ void k_split_rows(int64_t rows, int64_t rows_pad, int64_t K, int nkb, const uint16_t *__restrict__ A,
                             int64_t lda, uint8_t *__restrict__ lo, uint8_t *__restrict__ hi)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows_pad * KP * nkb) return;
    const int64_t i = idx / (KP * nkb), k = idx % (KP * nkb);
    const uint16_t v = (i < rows && k < K) ? A[i * lda + k] : 0;
    const size_t o = (size_t)((i / BM) * nkb + k / KP) * A_PLANE + tc::toff((uint32_t)(i % BM), (uint32_t)(k % KP));
    lo[o] = (uint8_t)(v & 0xff);
    hi[o] = (uint8_t)(v >> 8);
}

// K x cols (ldb) u16 -> B tiles (limb planes, K-major), zero padded; K-block i starts at
// i * cols_pad * KP (the multi-K GEMM's b_kb_stride)
__global__ void k_split_cols(int64_t cols, int64_t cols_pad, int64_t K, int nkb, const uint16_t *__restrict__ B,
                             int64_t ldb, uint8_t *__restrict__ lo, uint8_t *__restrict__ hi, Field F,
                             uint8_t *__restrict__ lo2, uint8_t *__restrict__ hi2)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= cols_pad * KP * nkb) return;
    const int64_t x = idx % cols_pad, k = idx / cols_pad;
    const uint16_t v = (x < cols && k < K) ? B[k * ldb + x] : 0;
    const size_t o = (size_t)(k / KP) * cols_pad * KP + (size_t)(x / BN) * B_PLANE +
                     toff64((uint32_t)(x % BN), (uint32_t)(k % KP));
    lo[o] = (uint8_t)(v & 0xff);
    hi[o] = (uint8_t)(v >> 8);
    if (lo2) {                                    // B' = 2^8 B mod p (multi-K pair kernel)
        const uint32_t w = fmod32((uint32_t)v << 8, F);
        lo2[o] = (uint8_t)(w & 0xff);
        hi2[o] = (uint8_t)(w >> 8);
    }
}

// a permutation of [0, n) for the K11 microbenchmark: i -> (a i + b) mod n with gcd(a, n) = 1
__global__ void k_bench_perm(int64_t n, uint32_t *__restrict__ perm)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t a = 2654435761ull % (uint64_t)n;
    if (a == 0) a = 1;
    auto g = [](uint64_t x, uint64_t y) { while (y) { const uint64_t t = x % y; x = y; y = t; } return x; };
    while (g(a, (uint64_t)n) != 1) a++;
    perm[i] = (uint32_t)((a * (uint64_t)i + 12345u) % (uint64_t)n);
}

// deterministic pseudo-random bytes / residues for the K11 microbenchmark
__global__ void k_fill_hash(uint8_t *__restrict__ p, size_t n, uint32_t seed)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u ^ seed;
        x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
        p[i] = (uint8_t)x;
    }
}
__global__ void k_fill_res(uint16_t *__restrict__ p, size_t n, uint32_t prime, uint32_t seed)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t x = (uint32_t)i * 2654435761u ^ seed;
        x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
        p[i] = (uint16_t)(x % prime);
    }
}

template <int MODE, int EPIW, bool PF2, bool MK = false>
gbla_status set_attr()
{
    static unsigned long long attr = 0;   // devices done (dev_bit)
    if (!(attr & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_modgemm_ws<MODE, EPIW, PF2, MK>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, ws_smem(MK)));
        attr |= dev_bit();
    }
    return GBLA_OK;
}

static int epi_warps()
{
    static int w = -1;
    if (w < 0) {
        const char *e = getenv("GBLA_EPI_WARPS");
        w = (e && atoi(e) == 16) ? 16 : 8;
    }
    return w;
}

static bool epi_pf2()
{
    static int v = -1;
    if (v < 0) v = getenv("GBLA_EPI_PF1") ? 0 : 1;
    return v == 1;
}

template <int MODE, int EPIW, bool PF2, bool MK = false>
static gbla_status launch_ws1(const MMArgs &a, int64_t grid, cudaStream_t st)
{
    GBLA_TRY((set_attr<MODE, EPIW, PF2, MK>()));
    // programmatic dependent launch: the GEMM's launch overlaps the tail of the previous kernel
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(ws_threads(EPIW));
    cfg.dynamicSmemBytes = ws_smem(MK);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    GBLA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_modgemm_ws<MODE, EPIW, PF2, MK>, a));
    return GBLA_OK;
}

template <int MODE>
static gbla_status launch_ws(const MMArgs &a, int64_t grid, cudaStream_t st)
{
    if (epi_warps() == 16) return epi_pf2() ? launch_ws1<MODE, 16, true>(a, grid, st) : launch_ws1<MODE, 16, false>(a, grid, st);
    return epi_pf2() ? launch_ws1<MODE, 8, true>(a, grid, st) : launch_ws1<MODE, 8, false>(a, grid, st);
}

int g_sms = 148;
// K11 multi-K on CTA pairs (k_modgemm_mk2, the default); GBLA_K11_PAIR=0 selects the single-CTA
// kernel (k_modgemm_ws<MK>), which needs no B' planes
static bool use_pair()
{
    static int v = -1;
    if (v < 0) v = (getenv("GBLA_K11_PAIR") && atoi(getenv("GBLA_K11_PAIR")) == 0) ? 0 : 1;
    return v == 1;
}

static gbla_status launch_pair(const MMArgs &a, int64_t max_rows, int64_t cols, int64_t grid, cudaStream_t st)
{
    static unsigned long long attr2 = 0;   // devices done (dev_bit)
    if (!(attr2 & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_modgemm_mk2, cudaFuncAttributeMaxDynamicSharedMemorySize, PR_SMEM));
        attr2 |= dev_bit();
    }
    const int64_t ptiles = ((max_rows + 2 * BM - 1) / (2 * BM)) * ((cols + PR_NP - 1) / PR_NP);
    int64_t pairs = grid / 2;
    if (pairs > ptiles) pairs = ptiles;
    if (pairs < 1) pairs = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    cfg.blockDim = dim3(ws_threads(8));
    cfg.dynamicSmemBytes = PR_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    GBLA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_modgemm_mk2, a));
    note_launch();
    return GBLA_OK;
}

int g_k11_exp = 0;       // gbla_modgemm_bench experiments (GBLA_K11_EXP; 0 everywhere else)

}  // namespace

// ---- host launchers used by echelon.cu -------------------------------------
// A tiles: rows grouped by 128 (A_PLANE bytes per plane per tile); B tiles:
// columns grouped by 64 (B_PLANE bytes per plane per tile).
gbla_status modgemm_tc_sub(cudaStream_t st, int64_t max_rows, const uint32_t *nrows_dev, int64_t cols, Field F,
                           const uint8_t *Alo, const uint8_t *Ahi, const uint8_t *Blo, const uint8_t *Bhi,
                           const uint32_t *rowidx, uint16_t *C, int64_t ldc, const int64_t *c0_dev,
                           const int64_t *win_dev, int64_t win_w, int ctsel, int grid_cap, const int64_t *cend_dev)
{
    if (max_rows <= 0 || cols <= 0) return GBLA_OK;
    const int64_t tiles = ((max_rows + BM - 1) / BM) * ((cols + BN - 1) / BN);
    int64_t grid = grid_cap > 0 ? grid_cap : g_sms;
    if (grid > tiles) grid = tiles;
    MMArgs a{max_rows, nrows_dev, cols, F, Alo, Ahi, Blo, Bhi, rowidx, C, ldc, nullptr, nullptr,
             c0_dev, nullptr, win_dev, win_w, ctsel, 1, 1, 0, nullptr, cend_dev, g_k11_exp};
    GBLA_TRY(launch_ws<MODE_SUB>(a, grid, st));
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

gbla_status modgemm_tc_store(cudaStream_t st, int64_t cols, Field F, const uint8_t *Alo, const uint8_t *Ahi,
                             const uint8_t *Blo, const uint8_t *Bhi, uint16_t *O, int64_t ldo, uint8_t *Tlo,
                             uint8_t *Thi, const int64_t *c0_dev, const uint32_t *skip_dev, const int64_t *win_dev,
                             int64_t win_w, int ctsel, const uint32_t *orows, int grid_cap, uint8_t *Tlo2,
                             uint8_t *Thi2)
{
    if (orows && (!skip_dev || !c0_dev)) { set_error("modgemm_tc_store: row map needs the pivot count"); return GBLA_E_INVAL; }
    if (cols <= 0) return GBLA_OK;
    const int64_t tiles = (cols + BN - 1) / BN;
    int64_t grid = (tiles + 1) / 2;                       // two column tiles per CTA (TMEM double buffer)
    if (grid > g_sms) grid = g_sms;
    if (grid_cap > 0 && grid > grid_cap) grid = grid_cap;
    MMArgs a{BM, nullptr, cols, F, Alo, Ahi, Blo, Bhi, orows, O, ldo, Tlo, Thi, c0_dev, skip_dev, win_dev, win_w, ctsel};
    a.Tlo2 = Tlo2;
    a.Thi2 = Thi2;
    GBLA_TRY(launch_ws<MODE_STORE>(a, grid, st));
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

// C[rowidx[i], c0:cols] -= sum over nkb K-blocks of A_i B_i (multi-K, K <= 512; see MMArgs)
gbla_status modgemm_tc_sub_mk(cudaStream_t st, int64_t max_rows, const uint32_t *nrows_dev, int64_t cols, Field F,
                              const uint8_t *Alo, const uint8_t *Ahi, int64_t a_rt_stride, int nkb,
                              const uint8_t *Blo, const uint8_t *Bhi, int64_t b_kb_stride, const int64_t *kb_c0,
                              const uint32_t *rowidx, uint16_t *C, int64_t ldc, const int64_t *c0_dev,
                              const int64_t *win_dev, int64_t win_w, int ctsel, int grid_cap, const uint8_t *B2lo,
                              const uint8_t *B2hi)
{
    if (max_rows <= 0 || cols <= 0 || nkb <= 0) return GBLA_OK;
    if (nkb > MK_MAX) { set_error("modgemm_tc_sub_mk: K > %d", MK_MAX * KP); return GBLA_E_INVAL; }
    const int64_t tiles = ((max_rows + BM - 1) / BM) * ((cols + BN - 1) / BN);
    int64_t grid = grid_cap > 0 ? grid_cap : g_sms;
    if (grid > tiles) grid = tiles;
    MMArgs a{max_rows, nrows_dev, cols, F, Alo, Ahi, Blo, Bhi, rowidx, C, ldc, nullptr, nullptr,
             c0_dev, nullptr, win_dev, win_w, ctsel, nkb, a_rt_stride, b_kb_stride, kb_c0, nullptr, g_k11_exp};
    // (up to 128 rows -- the super-panel fix-ups -- half of every pair would idle: one CTA per tile)
    if (use_pair() && B2lo && B2hi && max_rows > BM) {
        // CTA pairs over row-tile pairs: the A tiles of row tile 2 * ceil(rows / 256) - 1 are read
        // (zero rows: the caller's A buffer holds an even number of row tiles), and the B tiles of an
        // even number of 64-column tiles (the callers' B buffers are padded)
        a.B2lo = B2lo;
        a.B2hi = B2hi;
        return launch_pair(a, max_rows, cols, grid, st);
    }
    GBLA_TRY((launch_ws1<MODE_SUB, 8, true, true>(a, grid, st)));
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

// the echelon's window step in one launch (see k_modgemm_win)
gbla_status modgemm_tc_win(cudaStream_t st, int64_t cols, Field F, const uint8_t *Tlo, const uint8_t *Thi,
                           const uint8_t *Bglo, const uint8_t *Bghi, uint8_t *Rlo, uint8_t *Rhi,
                           const uint8_t *Flo, const uint8_t *Fhi, const uint32_t *rows, const uint32_t *sel,
                           const uint32_t *nrows_dev, const uint32_t *kp_dev, const int64_t *c0_dev,
                           const int64_t *win_dev, int64_t win_w, uint16_t *D, int64_t ldD, uint32_t *flags,
                           uint32_t epoch, int grid, uint8_t *Rlo2, uint8_t *Rhi2)
{
    static unsigned long long attr = 0;   // devices done (dev_bit)
    if (!(attr & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_modgemm_win, cudaFuncAttributeMaxDynamicSharedMemorySize, WS_SMEM));
        attr |= dev_bit();
    }
    WinArgs a{F, Tlo, Thi, Bglo, Bghi, Rlo, Rhi, Rlo2, Rhi2, Flo, Fhi, rows, sel, nrows_dev, kp_dev, c0_dev, win_dev,
              win_w, cols, D, ldD, flags, epoch};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(ws_threads(8));
    cfg.dynamicSmemBytes = WS_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    GBLA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_modgemm_win, a));
    note_launch();
    return GBLA_OK;
}

void modgemm_set_sms(int sms) { g_sms = sms > 0 ? sms : 148; }

// ---- C ABI: K11 as a standalone op -------------------------------------
// K <= 128: one K-block (k_modgemm_ws); 128 < K <= 512: the multi-K kernel of the deferred
// super-panel updates (exact: every limb sum <= 512 * 255^2 * 2 < 2^31).
static gbla_status modgemm_tiles(cudaStream_t st, const Field &F, int64_t rows, int64_t cols, int nkb,
                                 const uint8_t *Alo, const uint8_t *Ahi, const uint8_t *Blo, const uint8_t *Bhi,
                                 int64_t cp, const uint32_t *rowidx, uint16_t *C, int64_t ldc, const uint8_t *B2lo,
                                 const uint8_t *B2hi)
{
    if (nkb == 1 && !(getenv("GBLA_K11_K128_PAIR") && atoi(getenv("GBLA_K11_K128_PAIR")) == 1))
        return modgemm_tc_sub(st, rows, nullptr, cols, F, Alo, Ahi, Blo, Bhi, rowidx, C, ldc, nullptr, nullptr, 0,
                              CT_ALL, 0, nullptr);
    return modgemm_tc_sub_mk(st, rows, nullptr, cols, F, Alo, Ahi, nkb, nkb, Blo, Bhi, cp * KP, nullptr, rowidx, C,
                             ldc, nullptr, nullptr, 0, CT_ALL, 0, B2lo, B2hi);
}

extern "C" gbla_status gbla_modgemm(gbla_ctx ctx, uint32_t p, int64_t rows, int64_t cols, int64_t K,
                                    const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb,
                                    const uint32_t *rowidx, uint16_t *C, int64_t ldc, int engine, void *stream)
{
    if (!ctx || !A || !B || !C) { set_error("gbla_modgemm: NULL argument"); return GBLA_E_INVAL; }
    if (rows < 0 || cols < 0 || K < 0 || K > MK_MAX * KP || lda < K || ldb < cols || ldc < cols) {
        set_error("gbla_modgemm: bad sizes (K must be <= %d)", MK_MAX * KP);
        return GBLA_E_INVAL;
    }
    if (p <= 2 || p >= 65536) { set_error("gbla_modgemm: p out of range"); return GBLA_E_DOMAIN; }
    if (rows == 0 || cols == 0) return GBLA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    GBLA_CUDA_TRY(cudaSetDevice(ctx->device));
    modgemm_set_sms(ctx->sm_count);
    const Field F = make_field(p);
    if (engine == 1) {
        dim3 g(grid_for(cols, 128), (unsigned)rows);
        k_modgemm_int<<<g, 128, 0, st>>>(rows, cols, K, F, A, lda, B, ldb, rowidx, C, ldc);
        note_launch();
        GBLA_CUDA_TRY(cudaGetLastError());
        return GBLA_OK;
    }
    const int nkb = K <= KP ? 1 : (int)((K + KP - 1) / KP);
    const int64_t rp = (rows + 2 * BM - 1) / (2 * BM) * (2 * BM), cp = (cols + 2 * BN - 1) / (2 * BN) * (2 * BN);
    const size_t bytes = (size_t)(rp + 2 * cp) * KP * nkb * 2 + 256;
    uint8_t *ws = (uint8_t *)ctx_alloc(ctx, bytes, st);
    if (!ws) { set_error("gbla_modgemm: workspace allocation failed"); return GBLA_E_NOMEM; }
    uint8_t *Alo = ws, *Ahi = Alo + rp * KP * nkb, *Blo = Ahi + rp * KP * nkb, *Bhi = Blo + cp * KP * nkb;
    uint8_t *B2lo = Bhi + cp * KP * nkb, *B2hi = B2lo + cp * KP * nkb;
    k_split_rows<<<grid_for(rp * KP * nkb, 256), 256, 0, st>>>(rows, rp, K, nkb, A, lda, Alo, Ahi);
    k_split_cols<<<grid_for(cp * KP * nkb, 256), 256, 0, st>>>(cols, cp, K, nkb, B, ldb, Blo, Bhi, F, B2lo, B2hi);
    note_launch(2);
    gbla_status s = modgemm_tiles(st, F, rows, cols, nkb, Alo, Ahi, Blo, Bhi, cp, rowidx, C, ldc, B2lo, B2hi);
    cudaStreamSynchronize(st);
    ctx_free(ctx, ws, st);
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    return s;
}

// C[i, x] -= sum_{k < K} A[i, k] B[k, x] mod p for any K (f2's B'' = B' - B'[:, pivcol] R, K = rank):
// chunks of 512 through the multi-K CTA-pair kernel, workspace from the context allocator.
gbla_status modgemm_sub_chunked(gbla_ctx ctx, cudaStream_t st, const Field &F, int64_t rows, int64_t cols, int64_t K,
                                const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb, uint16_t *C, int64_t ldc)
{
    if (rows <= 0 || cols <= 0 || K <= 0) return GBLA_OK;
    modgemm_set_sms(ctx->sm_count);
    const int nkb = MK_MAX;
    const int64_t rp = (rows + 2 * BM - 1) / (2 * BM) * (2 * BM), cp = (cols + 2 * BN - 1) / (2 * BN) * (2 * BN);
    const size_t bytes = (size_t)(rp + 2 * cp) * KP * nkb * 2 + 256;
    uint8_t *ws = (uint8_t *)ctx_alloc(ctx, bytes, st);
    if (!ws) { set_error("modgemm_sub_chunked: workspace allocation of %zu bytes failed", bytes); return GBLA_E_NOMEM; }
    uint8_t *Alo = ws, *Ahi = Alo + rp * KP * nkb, *Blo = Ahi + rp * KP * nkb, *Bhi = Blo + cp * KP * nkb;
    uint8_t *B2lo = Bhi + cp * KP * nkb, *B2hi = B2lo + cp * KP * nkb;
    gbla_status s = GBLA_OK;
    for (int64_t k0 = 0; k0 < K && s == GBLA_OK; k0 += (int64_t)nkb * KP) {
        const int64_t kc = K - k0 < (int64_t)nkb * KP ? K - k0 : (int64_t)nkb * KP;
        k_split_rows<<<grid_for(rp * KP * nkb, 256), 256, 0, st>>>(rows, rp, kc, nkb, A + k0, lda, Alo, Ahi);
        k_split_cols<<<grid_for(cp * KP * nkb, 256), 256, 0, st>>>(cols, cp, kc, nkb, B + (size_t)k0 * ldb, ldb, Blo,
                                                                  Bhi, F, B2lo, B2hi);
        note_launch(2);
        s = modgemm_tc_sub_mk(st, rows, nullptr, cols, F, Alo, Ahi, nkb, nkb, Blo, Bhi, cp * KP, nullptr, nullptr, C,
                              ldc, nullptr, nullptr, 0, CT_ALL, 0, B2lo, B2hi);
        if (s == GBLA_OK && cudaGetLastError() != cudaSuccess) { set_error("modgemm_sub_chunked: launch failed"); s = GBLA_E_CUDA; }
    }
    ctx_free(ctx, ws, st);
    return s;
}

// K11 microbenchmark: random operand tiles and C (rows x cols, K = 128 * nkb) on the device,
// one untimed launch, then `reps` launches timed with CUDA events on `stream`.
extern "C" gbla_status gbla_modgemm_bench(gbla_ctx ctx, uint32_t p, int64_t rows, int64_t cols, int64_t K, int reps,
                                          void *stream, float *ms_per_launch)
{
    if (!ctx || !ms_per_launch || rows <= 0 || cols <= 0 || K <= 0 || K > MK_MAX * KP || reps <= 0) {
        set_error("gbla_modgemm_bench: bad arguments");
        return GBLA_E_INVAL;
    }
    if (p <= 2 || p >= 65536) { set_error("gbla_modgemm_bench: p out of range"); return GBLA_E_DOMAIN; }
    cudaStream_t st = (cudaStream_t)stream;
    GBLA_CUDA_TRY(cudaSetDevice(ctx->device));
    modgemm_set_sms(ctx->sm_count);
    const Field F = make_field(p);
    const int nkb = (int)((K + KP - 1) / KP);
    const int64_t rp = (rows + 2 * BM - 1) / (2 * BM) * (2 * BM), cp = (cols + 2 * BN - 1) / (2 * BN) * (2 * BN), ldc = cp;
    const size_t opb = (size_t)(rp + 2 * cp) * KP * nkb * 2, cb = (size_t)rows * ldc * 2;
    uint8_t *ws = (uint8_t *)ctx_alloc(ctx, opb + cb + 256, st);
    if (!ws) { set_error("gbla_modgemm_bench: allocation failed"); return GBLA_E_NOMEM; }
    uint8_t *Alo = ws, *Ahi = Alo + rp * KP * nkb, *Blo = Ahi + rp * KP * nkb, *Bhi = Blo + cp * KP * nkb;
    uint8_t *B2lo = Bhi + cp * KP * nkb, *B2hi = B2lo + cp * KP * nkb;
    uint16_t *C = reinterpret_cast<uint16_t *>(ws + (opb + 255) / 256 * 256);
    // GBLA_K11_BENCH_PERM=1: C rows gathered through a pseudo-random row index (the echelon's
    // flushes address D rows in lead order, scattered in memory)
    uint32_t *perm = nullptr;
    if (getenv("GBLA_K11_BENCH_PERM") && atoi(getenv("GBLA_K11_BENCH_PERM")) == 1) {
        perm = (uint32_t *)ctx_alloc(ctx, (size_t)rows * 4 + 16, st);
        if (!perm) { ctx_free(ctx, ws, st); set_error("gbla_modgemm_bench: allocation failed"); return GBLA_E_NOMEM; }
        k_bench_perm<<<grid_for(rows, 256), 256, 0, st>>>(rows, perm);
    }
    k_fill_hash<<<4 * ctx->sm_count, 256, 0, st>>>(ws, opb, 12345u);
    k_fill_res<<<4 * ctx->sm_count, 256, 0, st>>>(C, (size_t)rows * ldc, p, 777u);
    note_launch(2);
    gbla_status s = modgemm_tiles(st, F, rows, cols, nkb, Alo, Ahi, Blo, Bhi, cp, perm, C, ldc, B2lo, B2hi);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (s == GBLA_OK && (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)) {
        set_error("gbla_modgemm_bench: event creation failed");
        s = GBLA_E_CUDA;
    }
    if (s == GBLA_OK) {
        g_k11_exp = getenv("GBLA_K11_EXP") ? atoi(getenv("GBLA_K11_EXP")) : 0;
        cudaEventRecord(e0, st);
        for (int r = 0; r < reps && s == GBLA_OK; r++)
            s = modgemm_tiles(st, F, rows, cols, nkb, Alo, Ahi, Blo, Bhi, cp, perm, C, ldc, B2lo, B2hi);
        cudaEventRecord(e1, st);
        g_k11_exp = 0;
        if (cudaEventSynchronize(e1) != cudaSuccess) { set_error("gbla_modgemm_bench: kernel failed"); s = GBLA_E_CUDA; }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        *ms_per_launch = ms / reps;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaStreamSynchronize(st);
    ctx_free(ctx, ws, st);
    if (perm) ctx_free(ctx, perm, st);
    cudaGetLastError();
    return s;
}
