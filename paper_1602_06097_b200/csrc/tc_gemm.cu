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
// Tile: BM = 128 rows (TMEM lanes) x BN = 64 columns, K = 128.  TMEM holds
// three accumulators HH | X | LL (3 x 64 columns of a 256-column
// allocation).  One thread issues 16 MMAs (4 K-steps of 32 x 4 limb
// products), commits to an mbarrier; 4 warps run the epilogue
// (tcgen05.ld 32x32b: warp w owns lanes 32w..32w+31).
//   MODE_SUB    C[rowidx[i], x] = C - S   mod p     (trailing update)
//   MODE_STORE  O[i, x] = S mod p, plus the transposed limb planes of O
//               (the B operand of a following MODE_SUB GEMM)
#include "internal.cuh"
#include "tc.cuh"

namespace {

constexpr int BM = 128, BN = 64, KP = 128;
constexpr int SMEM_A = BM * KP;     // bytes per limb plane
constexpr int SMEM_B = BN * KP;
constexpr int SMEM_TOTAL = 2 * SMEM_A + 2 * SMEM_B;
enum { MODE_SUB = 0, MODE_STORE = 1 };

template <int MODE>
__global__ void __launch_bounds__(128) k_modgemm_tc(
    int64_t nrows, const uint32_t *__restrict__ nrows_dev, int64_t cols, Field F,
    const uint8_t *__restrict__ Alo, const uint8_t *__restrict__ Ahi,     // [rows_pad][KP]
    const uint8_t *__restrict__ Blo, const uint8_t *__restrict__ Bhi,     // [cols_pad][KP]
    const uint32_t *__restrict__ rowidx, uint16_t *__restrict__ C, int64_t ldc,
    uint8_t *__restrict__ Tlo, uint8_t *__restrict__ Thi,                 // MODE_STORE: [cols_pad][KP]
    bool vec)                                                             // C rows 32-byte aligned
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sAh = smem, *sAl = smem + SMEM_A, *sBh = smem + 2 * SMEM_A, *sBl = smem + 2 * SMEM_A + SMEM_B;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int64_t nr = nrows_dev ? (int64_t)*nrows_dev : nrows;
    const int64_t row0 = (int64_t)blockIdx.y * BM;
    const int64_t x0 = (int64_t)blockIdx.x * BN;
    if (row0 >= nr || x0 >= cols) return;
    const int tid = threadIdx.x, warp = tid >> 5;

    if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
    if (tid == 0) tc::mbar_init(&bar, 1);

    // A tile -> core-matrix layout: chunk (row r, k16 q) at q*BM*16 + (r/8)*128 + (r%8)*16
    for (int i = tid; i < BM * (KP / 16); i += 128) {
        const int r = i >> 3, q = i & 7;
        uint4 vh = make_uint4(0, 0, 0, 0), vl = vh;
        if (row0 + r < nr) {
            const size_t g = (size_t)(row0 + r) * KP + q * 16;
            vh = *reinterpret_cast<const uint4 *>(Ahi + g);
            vl = *reinterpret_cast<const uint4 *>(Alo + g);
        }
        const int o = q * (BM * 16) + (r >> 3) * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4 *>(sAh + o) = vh;
        *reinterpret_cast<uint4 *>(sAl + o) = vl;
    }
    for (int i = tid; i < BN * (KP / 16); i += 128) {
        const int x = i >> 3, q = i & 7;
        uint4 vh = make_uint4(0, 0, 0, 0), vl = vh;
        if (x0 + x < cols) {
            const size_t g = (size_t)(x0 + x) * KP + q * 16;
            vh = *reinterpret_cast<const uint4 *>(Bhi + g);
            vl = *reinterpret_cast<const uint4 *>(Blo + g);
        }
        const int o = q * (BN * 16) + (x >> 3) * 128 + (x & 7) * 16;
        *reinterpret_cast<uint4 *>(sBh + o) = vh;
        *reinterpret_cast<uint4 *>(sBl + o) = vl;
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_base;

    if (tid == 0) {
        const uint32_t idesc = tc::idesc_u8(BM, BN);
        const uint32_t aH = tc::smem_u32(sAh), aL = tc::smem_u32(sAl);
        const uint32_t bH = tc::smem_u32(sBh), bL = tc::smem_u32(sBl);
#pragma unroll
        for (int s = 0; s < KP / 32; s++) {
            const uint32_t ao = s * 2 * (BM * 16), bo = s * 2 * (BN * 16);
            const uint64_t dAh = tc::desc_kmajor(aH + ao, BM * 16, 128);
            const uint64_t dAl = tc::desc_kmajor(aL + ao, BM * 16, 128);
            const uint64_t dBh = tc::desc_kmajor(bH + bo, BN * 16, 128);
            const uint64_t dBl = tc::desc_kmajor(bL + bo, BN * 16, 128);
            tc::mma_i8(tbase + 0, dAh, dBh, idesc, s > 0);          // HH
            tc::mma_i8(tbase + BN, dAh, dBl, idesc, s > 0);         // X
            tc::mma_i8(tbase + BN, dAl, dBh, idesc, 1);             // X
            tc::mma_i8(tbase + 2 * BN, dAl, dBl, idesc, s > 0);     // LL
        }
        tc::commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after();

    // epilogue: thread tid <-> tile row tid <-> TMEM lane tid
    const int64_t slot = row0 + tid;
    const bool live = slot < nr;
    const uint32_t lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
    uint16_t *crow = nullptr;
    if (live) crow = C + (size_t)(MODE == MODE_SUB && rowidx ? rowidx[slot] : slot) * ldc + x0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
        uint32_t hh[16], xx[16], ll[16];
        tc::tmem_ld16(lane_addr + c, hh);
        tc::tmem_ld16(lane_addr + BN + c, xx);
        tc::tmem_ld16(lane_addr + 2 * BN + c, ll);
        tc::tmem_wait_ld();
        if (!live) continue;
        if (vec && x0 + c + 16 <= cols) {
            // 32-byte row segments: two 16-byte vector accesses per chunk
            uint4 v[2];
            uint16_t *d = reinterpret_cast<uint16_t *>(v);
            if (MODE == MODE_SUB) {
                v[0] = *reinterpret_cast<const uint4 *>(crow + c);
                v[1] = *reinterpret_cast<const uint4 *>(crow + c + 8);
            }
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint64_t S = ((uint64_t)hh[j] << 16) + ((uint64_t)xx[j] << 8) + ll[j];
                const uint32_t s = fmod64(S, F);
                if (MODE == MODE_SUB) {
                    const uint32_t dv = d[j];
                    d[j] = (uint16_t)(dv >= s ? dv - s : dv + F.p - s);
                } else {
                    d[j] = (uint16_t)s;
                    const int64_t x = x0 + c + j;
                    Tlo[(size_t)x * KP + slot] = (uint8_t)(s & 0xff);
                    Thi[(size_t)x * KP + slot] = (uint8_t)(s >> 8);
                }
            }
            *reinterpret_cast<uint4 *>(crow + c) = v[0];
            *reinterpret_cast<uint4 *>(crow + c + 8) = v[1];
            continue;
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int64_t x = x0 + c + j;
            if (x >= cols) break;
            const uint64_t S = ((uint64_t)hh[j] << 16) + ((uint64_t)xx[j] << 8) + ll[j];
            const uint32_t s = fmod64(S, F);
            if (MODE == MODE_SUB) {
                const uint32_t d = crow[c + j];
                crow[c + j] = (uint16_t)(d >= s ? d - s : d + F.p - s);
            } else {
                crow[c + j] = (uint16_t)s;
                Tlo[(size_t)x * KP + slot] = (uint8_t)(s & 0xff);
                Thi[(size_t)x * KP + slot] = (uint8_t)(s >> 8);
            }
        }
    }
    tc::fence_before();
    __syncthreads();
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

// rows x K (lda) u16 -> limb planes [rows_pad][KP], zero padded
__global__ void k_split_rows(int64_t rows, int64_t rows_pad, int64_t K, const uint16_t *__restrict__ A, int64_t lda,
                             uint8_t *__restrict__ lo, uint8_t *__restrict__ hi)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows_pad * KP) return;
    const int64_t i = idx / KP, k = idx % KP;
    const uint16_t v = (i < rows && k < K) ? A[i * lda + k] : 0;
    lo[idx] = (uint8_t)(v & 0xff);
    hi[idx] = (uint8_t)(v >> 8);
}

// K x cols (ldb) u16 -> transposed limb planes [cols_pad][KP], zero padded
__global__ void k_split_cols(int64_t cols, int64_t cols_pad, int64_t K, const uint16_t *__restrict__ B, int64_t ldb,
                             uint8_t *__restrict__ lo, uint8_t *__restrict__ hi)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= cols_pad * KP) return;
    const int64_t x = idx / KP, k = idx % KP;
    const uint16_t v = (x < cols && k < K) ? B[k * ldb + x] : 0;
    lo[idx] = (uint8_t)(v & 0xff);
    hi[idx] = (uint8_t)(v >> 8);
}

}  // namespace

// host launchers used by echelon.cu
gbla_status modgemm_tc_sub(cudaStream_t st, int64_t max_rows, const uint32_t *nrows_dev, int64_t cols, Field F,
                           const uint8_t *Alo, const uint8_t *Ahi, const uint8_t *Blo, const uint8_t *Bhi,
                           const uint32_t *rowidx, uint16_t *C, int64_t ldc)
{
    static bool attr = false;
    if (!attr) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_modgemm_tc<MODE_SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           SMEM_TOTAL));
        attr = true;
    }
    if (max_rows <= 0 || cols <= 0) return GBLA_OK;
    dim3 grid(grid_for(cols, BN), grid_for(max_rows, BM));
    const bool vec = ((reinterpret_cast<uintptr_t>(C) & 31) == 0) && (ldc % 16 == 0);
    k_modgemm_tc<MODE_SUB><<<grid, 128, SMEM_TOTAL, st>>>(max_rows, nrows_dev, cols, F, Alo, Ahi, Blo, Bhi, rowidx,
                                                          C, ldc, nullptr, nullptr, vec);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

gbla_status modgemm_tc_store(cudaStream_t st, int64_t cols, Field F, const uint8_t *Alo, const uint8_t *Ahi,
                             const uint8_t *Blo, const uint8_t *Bhi, uint16_t *O, int64_t ldo, uint8_t *Tlo,
                             uint8_t *Thi)
{
    static bool attr = false;
    if (!attr) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_modgemm_tc<MODE_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           SMEM_TOTAL));
        attr = true;
    }
    if (cols <= 0) return GBLA_OK;
    dim3 grid(grid_for(cols, BN), 1);
    const bool vec = ((reinterpret_cast<uintptr_t>(O) & 31) == 0) && (ldo % 16 == 0);
    k_modgemm_tc<MODE_STORE><<<grid, 128, SMEM_TOTAL, st>>>(BM, nullptr, cols, F, Alo, Ahi, Blo, Bhi, nullptr, O, ldo,
                                                            Tlo, Thi, vec);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

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
    gbla_status s = modgemm_tc_sub(st, rows, nullptr, cols, F, Alo, Ahi, Blo, Bhi, rowidx, C, ldc);
    cudaStreamSynchronize(st);
    ctx_free(ctx, ws, st);
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    return s;
}
