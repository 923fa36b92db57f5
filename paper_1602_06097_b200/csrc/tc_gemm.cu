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
// Persistent kernel: CTA b (128 threads) owns a contiguous range of output
// tiles (BM = 128 rows x BN = 64 columns) in row-tile-major order, so the A
// tile of a row tile is fetched once and reused for all of its column tiles
// (a stage re-copies A only when its row tile changes); the next tile's
// operands are double-buffered behind the current MMAs.  TMEM holds
// HH | X | LL (3 x 64 columns of a 256-column allocation); one thread issues
// 16 MMAs (4 K-steps x 4 limb products) and commits to an mbarrier; 4 warps
// run the epilogue: tcgen05.ld (warp w owns lanes 32w..32w+31), reduce mod
// p, stage the 128 x 64 result in shared memory (XOR-swizzled 16-byte
// chunks), then read-modify-write C one full 128-byte row segment per warp
// instruction.
//   MODE_SUB    C[rowidx[i], x] = C - S   mod p     (trailing update)
//   MODE_STORE  O[i, x] = S mod p, plus O's limb planes as B tiles
//               (the B operand of a following MODE_SUB GEMM)
#include "internal.cuh"
#include "tc.cuh"

namespace {

constexpr int BM = 128, BN = 64, KP = 128;
constexpr uint32_t A_PLANE = BM * KP;      // 16 KB
constexpr uint32_t B_PLANE = BN * KP;      // 8 KB
constexpr uint32_t A_BYTES = 2 * A_PLANE, B_BYTES = 2 * B_PLANE;
constexpr uint32_t STAGE = A_BYTES + B_BYTES;   // 48 KB
constexpr int SMEM_TOTAL = 2 * STAGE;
enum { MODE_SUB = 0, MODE_STORE = 1 };

using tc::toff64;


template <int MODE>
__global__ void __launch_bounds__(128) k_modgemm_tc(
    int64_t nrows, const uint32_t *__restrict__ nrows_dev, int64_t cols, Field F,
    const uint8_t *__restrict__ Alo, const uint8_t *__restrict__ Ahi,     // A tiles (row tile rt at rt*A_PLANE)
    const uint8_t *__restrict__ Blo, const uint8_t *__restrict__ Bhi,     // B tiles (col tile ct at ct*B_PLANE)
    const uint32_t *__restrict__ rowidx, uint16_t *__restrict__ C, int64_t ldc,
    uint8_t *__restrict__ Tlo, uint8_t *__restrict__ Thi,                 // MODE_STORE: output B tiles
    const int64_t *__restrict__ c0_dev,      // optional: columns [*c0_dev, cols) (MODE_SUB: of C)
    const uint32_t *__restrict__ skip_dev)   // optional: nothing to do when *skip_dev == 0
{
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[2], accbar;
    __shared__ uint32_t tmem_base;
    if (skip_dev && *skip_dev == 0) return;
    if (c0_dev) {
        const int64_t c0 = *c0_dev;
        cols -= c0;
        if (MODE == MODE_SUB) C += c0;
    }
    const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : nrows;
    const int64_t ntr = (nr + BM - 1) / BM, ntc = (cols + BN - 1) / BN, ntiles = ntr * ntc;
    const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t_begin = (int64_t)blockIdx.x * per;
    const int64_t t_end = t_begin + per < ntiles ? t_begin + per : ntiles;
    if (t_begin >= t_end) return;
    const int tid = threadIdx.x, warp = tid >> 5;
    const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && (ldc % 8 == 0);   // 16-byte row segments

    if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
    if (tid == 0) {
        tc::mbar_init(&full[0], 1);
        tc::mbar_init(&full[1], 1);
        tc::mbar_init(&accbar, 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_base;
    const uint32_t lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
    const uint32_t s0 = tc::smem_u32(smem);
    int64_t stage_rt[2] = {-1, -1};                     // row tile whose A is in each stage (thread 0)

    auto load = [&](int64_t tile, int s) {
        const int64_t rt = tile / ntc, ct = tile % ntc;
        uint8_t *st = smem + s * STAGE;
        const bool needA = stage_rt[s] != rt;
        tc::mbar_expect_tx(&full[s], needA ? STAGE : B_BYTES);
        if (needA) {
            tc::bulk_g2s(st, Ahi + rt * A_PLANE, A_PLANE, &full[s]);
            tc::bulk_g2s(st + A_PLANE, Alo + rt * A_PLANE, A_PLANE, &full[s]);
            stage_rt[s] = rt;
        }
        tc::bulk_g2s(st + A_BYTES, Bhi + ct * B_PLANE, B_PLANE, &full[s]);
        tc::bulk_g2s(st + A_BYTES + B_PLANE, Blo + ct * B_PLANE, B_PLANE, &full[s]);
    };
    if (tid == 0) load(t_begin, 0);
    uint32_t ph_full[2] = {0, 0}, ph_acc = 0;
    int s = 0;
    for (int64_t tile = t_begin; tile < t_end; tile++, s ^= 1) {
        const int64_t rt = tile / ntc, ct = tile % ntc;
        const int64_t row0 = rt * BM, x0 = ct * BN;
        if (tid == 0) {
            if (tile + 1 < t_end) load(tile + 1, s ^ 1);   // stage s^1 is free: its MMAs completed last iteration
            tc::mbar_wait(&full[s], ph_full[s]);
            tc::fence_after();
            const uint32_t idesc = tc::idesc_u8(BM, BN);
            const uint32_t aH = s0 + s * STAGE, aL = aH + A_PLANE, bH = aH + A_BYTES, bL = bH + B_PLANE;
#pragma unroll
            for (int k = 0; k < KP / 32; k++) {
                const uint32_t ao = k * 2 * (BM * 16), bo = k * 2 * (BN * 16);
                const uint64_t dAh = tc::desc_kmajor(aH + ao, BM * 16, 128);
                const uint64_t dAl = tc::desc_kmajor(aL + ao, BM * 16, 128);
                const uint64_t dBh = tc::desc_kmajor(bH + bo, BN * 16, 128);
                const uint64_t dBl = tc::desc_kmajor(bL + bo, BN * 16, 128);
                tc::mma_i8(tbase + 0, dAh, dBh, idesc, k > 0);          // HH
                tc::mma_i8(tbase + BN, dAh, dBl, idesc, k > 0);         // X
                tc::mma_i8(tbase + BN, dAl, dBh, idesc, 1);             // X
                tc::mma_i8(tbase + 2 * BN, dAl, dBl, idesc, k > 0);     // LL
            }
            tc::commit(&accbar);
        }
        ph_full[s] ^= 1;
        tc::mbar_wait(&accbar, ph_acc);
        ph_acc ^= 1;
        tc::fence_after();

        // epilogue: thread tid = tile row tid; its 128-byte row segment of C is
        // loaded first (8 vector loads in flight), the 4 TMEM chunks are folded in
        // (constant register indices: no local memory), then stored back
        const int64_t slot = row0 + tid;
        const bool live = slot < nr;
        uint16_t *crow = live ? C + (size_t)(MODE == MODE_SUB && rowidx ? rowidx[slot] : slot) * ldc + x0 : nullptr;
        const bool fast = live && vec && x0 + BN <= cols;
        uint32_t d[BN / 2];                                   // u16 pairs
#pragma unroll
        for (int w = 0; w < BN / 2; w++) d[w] = 0;
        if (MODE == MODE_SUB && live) {
            if (fast) {
#pragma unroll
                for (int u = 0; u < BN / 8; u++) {
                    const uint4 q = reinterpret_cast<const uint4 *>(crow)[u];
                    d[4 * u] = q.x; d[4 * u + 1] = q.y; d[4 * u + 2] = q.z; d[4 * u + 3] = q.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < BN; j++)
                    if (x0 + j < cols) d[j / 2] |= (uint32_t)crow[j] << (16 * (j & 1));
            }
        }
#pragma unroll
        for (int c = 0; c < BN; c += 16) {
            uint32_t hh[16], xx[16], ll[16];
            __syncwarp();
            tc::tmem_ld16(lane_addr + c, hh);
            tc::tmem_ld16(lane_addr + BN + c, xx);
            tc::tmem_ld16(lane_addr + 2 * BN + c, ll);
            tc::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
                const uint32_t s0 = fmod64(((uint64_t)hh[j] << 16) + ((uint64_t)xx[j] << 8) + ll[j], F);
                const uint32_t s1 = fmod64(((uint64_t)hh[j + 1] << 16) + ((uint64_t)xx[j + 1] << 8) + ll[j + 1], F);
                const int w = (c + j) / 2;
                if (MODE == MODE_SUB) {
                    uint32_t lo = d[w] & 0xffffu, hi = d[w] >> 16;
                    lo = lo >= s0 ? lo - s0 : lo + F.p - s0;
                    hi = hi >= s1 ? hi - s1 : hi + F.p - s1;
                    d[w] = lo | (hi << 16);
                } else {
                    d[w] = s0 | (s1 << 16);
                    // B tile planes of the result: row (= K index) slot, columns x (= MN index)
                    const uint32_t x = (uint32_t)(x0 + c + j);
                    const size_t o = (size_t)(x / BN) * B_PLANE + toff64(x % BN, (uint32_t)slot);
                    Tlo[o] = (uint8_t)(s0 & 0xff);
                    Thi[o] = (uint8_t)(s0 >> 8);
                    Tlo[o + 16] = (uint8_t)(s1 & 0xff);         // x+1 -> next core-matrix row (16 bytes on)
                    Thi[o + 16] = (uint8_t)(s1 >> 8);
                }
            }
        }
        tc::fence_before();
        __syncthreads();                  // TMEM free for the next tile's MMAs
        tc::fence_after();
        if (fast) {
#pragma unroll
            for (int u = 0; u < BN / 8; u++)
                reinterpret_cast<uint4 *>(crow)[u] = make_uint4(d[4 * u], d[4 * u + 1], d[4 * u + 2], d[4 * u + 3]);
        } else if (live) {
#pragma unroll
            for (int j = 0; j < BN; j++)
                if (x0 + j < cols) crow[j] = (uint16_t)(d[j / 2] >> (16 * (j & 1)));
        }
    }
    if (warp == 0) tc::tmem_dealloc<256>(tbase);
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

// rows x K (lda) u16 -> A tiles (limb planes), zero padded
__global__ void k_split_rows(int64_t rows, int64_t rows_pad, int64_t K, const uint16_t *__restrict__ A, int64_t lda,
                             uint8_t *__restrict__ lo, uint8_t *__restrict__ hi)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows_pad * KP) return;
    const int64_t i = idx / KP, k = idx % KP;
    const uint16_t v = (i < rows && k < K) ? A[i * lda + k] : 0;
    const size_t o = (size_t)(i / BM) * A_PLANE + tc::toff((uint32_t)(i % BM), (uint32_t)k);
    lo[o] = (uint8_t)(v & 0xff);
    hi[o] = (uint8_t)(v >> 8);
}

// K x cols (ldb) u16 -> B tiles (limb planes, K-major), zero padded
__global__ void k_split_cols(int64_t cols, int64_t cols_pad, int64_t K, const uint16_t *__restrict__ B, int64_t ldb,
                             uint8_t *__restrict__ lo, uint8_t *__restrict__ hi)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= cols_pad * KP) return;
    const int64_t x = idx % cols_pad, k = idx / cols_pad;
    const uint16_t v = (x < cols && k < K) ? B[k * ldb + x] : 0;
    const size_t o = (size_t)(x / BN) * B_PLANE + toff64((uint32_t)(x % BN), (uint32_t)k);
    lo[o] = (uint8_t)(v & 0xff);
    hi[o] = (uint8_t)(v >> 8);
}

template <int MODE>
gbla_status set_attr()
{
    static bool attr = false;
    if (!attr) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_modgemm_tc<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           SMEM_TOTAL));
        attr = true;
    }
    return GBLA_OK;
}

int g_sms = 148;

}  // namespace

// ---- host launchers used by echelon.cu -------------------------------------
// A tiles: rows grouped by 128 (A_PLANE bytes per plane per tile); B tiles:
// columns grouped by 64 (B_PLANE bytes per plane per tile).
gbla_status modgemm_tc_sub(cudaStream_t st, int64_t max_rows, const uint32_t *nrows_dev, int64_t cols, Field F,
                           const uint8_t *Alo, const uint8_t *Ahi, const uint8_t *Blo, const uint8_t *Bhi,
                           const uint32_t *rowidx, uint16_t *C, int64_t ldc, const int64_t *c0_dev)
{
    GBLA_TRY(set_attr<MODE_SUB>());
    if (max_rows <= 0 || cols <= 0) return GBLA_OK;
    const int64_t tiles = ((max_rows + BM - 1) / BM) * ((cols + BN - 1) / BN);
    const int64_t grid = tiles < 2 * g_sms ? tiles : 2 * g_sms;
    k_modgemm_tc<MODE_SUB><<<(unsigned)grid, 128, SMEM_TOTAL, st>>>(max_rows, nrows_dev, cols, F, Alo, Ahi, Blo, Bhi,
                                                                    rowidx, C, ldc, nullptr, nullptr, c0_dev, nullptr);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

gbla_status modgemm_tc_store(cudaStream_t st, int64_t cols, Field F, const uint8_t *Alo, const uint8_t *Ahi,
                             const uint8_t *Blo, const uint8_t *Bhi, uint16_t *O, int64_t ldo, uint8_t *Tlo,
                             uint8_t *Thi, const int64_t *c0_dev, const uint32_t *skip_dev)
{
    GBLA_TRY(set_attr<MODE_STORE>());
    if (cols <= 0) return GBLA_OK;
    const int64_t tiles = (cols + BN - 1) / BN;
    const int64_t grid = tiles < 2 * g_sms ? tiles : 2 * g_sms;
    k_modgemm_tc<MODE_STORE><<<(unsigned)grid, 128, SMEM_TOTAL, st>>>(BM, nullptr, cols, F, Alo, Ahi, Blo, Bhi,
                                                                      nullptr, O, ldo, Tlo, Thi, c0_dev, skip_dev);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

void modgemm_set_sms(int sms) { g_sms = sms > 0 ? sms : 148; }

// ---- C ABI: K11 as a standalone op -------------------------------------
extern "C" gbla_status gbla_modgemm(gbla_ctx ctx, uint32_t p, int64_t rows, int64_t cols, int64_t K,
                                    const uint16_t *A, int64_t lda, const uint16_t *B, int64_t ldb,
                                    const uint32_t *rowidx, uint16_t *C, int64_t ldc, int engine, void *stream)
{
    if (!ctx || !A || !B || !C) { set_error("gbla_modgemm: NULL argument"); return GBLA_E_INVAL; }
    if (rows < 0 || cols < 0 || K < 0 || K > KP || lda < K || ldb < cols || ldc < cols) {
        set_error("gbla_modgemm: bad sizes (K must be <= %d)", KP);
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
    const int64_t rp = (rows + BM - 1) / BM * BM, cp = (cols + BN - 1) / BN * BN;
    const size_t bytes = (size_t)(rp + cp) * KP * 2 + 256;
    uint8_t *ws = (uint8_t *)ctx_alloc(ctx, bytes, st);
    if (!ws) { set_error("gbla_modgemm: workspace allocation failed"); return GBLA_E_NOMEM; }
    uint8_t *Alo = ws, *Ahi = Alo + rp * KP, *Blo = Ahi + rp * KP, *Bhi = Blo + cp * KP;
    k_split_rows<<<grid_for(rp * KP, 256), 256, 0, st>>>(rows, rp, K, A, lda, Alo, Ahi);
    k_split_cols<<<grid_for(cp * KP, 256), 256, 0, st>>>(cols, cp, K, B, ldb, Blo, Bhi);
    note_launch(2);
    gbla_status s = modgemm_tc_sub(st, rows, nullptr, cols, F, Alo, Ahi, Blo, Bhi, rowidx, C, ldc, nullptr);
    cudaStreamSynchronize(st);
    ctx_free(ctx, ws, st);
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    return s;
}
