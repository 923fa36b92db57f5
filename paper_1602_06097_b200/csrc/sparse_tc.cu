// sparse_tc.cu -- the sparse triangular phase on the tensor cores.
//
// C' = C A^-1 and D_new = D - C' B, the 4-step variant of the new order
// ("carry out the reduction of C by A, but store the
// corresponding coefficients", then "reduce D by B using the coefficients
// stored in C'"), blocked by 128 x 128 tiles in sigma order:
//
//   band tiles   [A|B] rows in blocks I of 128 pivots; every 128 x 128 tile
//                of the band (A tiles J in [I, amax(I)], B tiles K in
//                [bmin(I), bmax(I)]) is stored DENSE as two u8 limb planes in
//                the tcgen05 K-major core-matrix layout, transposed (K = the
//                pivot index i, MN = the column): the B operand of X_I * A_IJ
//                and X_I * B_IK.  Padded pivots npiv..NB*128-1 are identity.
//   diag inverse inv(A_JJ) (unit upper triangular) per block, same layout.
//   K5' sweep    one CTA per tile T of 128 targets (sorted by lead), J
//                ascending from the tile's first lead block:
//                  Y   = C_J[T] - sum_{I<J, A_IJ != 0} X_I[T] A_IJ   (GEMM)
//                  X_J = Y inv(A_JJ)                                 (GEMM)
//                which is forward substitution x_t A = c_t (Alg 2) done a
//                block of 128 pivots at a time.  X_J[T] is stored as limb
//                planes (A operand of later steps and of the update).
//   K7' update   D[T, K] -= sum_I X_I[T] B_IK   (output-stationary GEMM)
// Every GEMM: tcgen05.mma kind::i8, M = N = 128, K = 128 per tile pair,
// three s32 TMEM accumulators HH | X | LL (exactness: tc_gemm.cu header),
// operands staged by cp.async.bulk (TMA bulk copies) in a 2-stage mbarrier
// pipeline, one elected thread issuing.  The results are the same exact
// residues as Alg 2 (X = C A^-1 is unique), bit for bit.
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include <cub/cub.cuh>

#include "internal.cuh"
#include "tc.cuh"

GBLA_DEV_ERR_UNIT(sweep_dev_err)

struct BandTiles {
    int64_t NB = 0, NNB = 0, ntiles = 0;
    int64_t nA = 0, nB = 0;
    uint8_t *tilesA = nullptr, *tilesB = nullptr, *invT = nullptr, *Xt = nullptr;
    uint64_t *offA = nullptr, *offB = nullptr;
    uint32_t *amax = nullptr, *bmin = nullptr, *bmax = nullptr;
    uint32_t *jl_ptr = nullptr, *jl_idx = nullptr, *kl_ptr = nullptr, *kl_idx = nullptr;
    unsigned long long *ops = nullptr;   // [3] A-part, B-part modMACs (Alg 2 count), tile pairs swept
    int64_t xt_cap = 0;                  // target tiles the X-tile buffer holds
    bool swept = false;
};

namespace {

constexpr uint32_t TB = 32768, PB = 16384;
// u8 MACs the tensor cores execute per tile pair of the sweep: 4 limb products of 128 x 128 x 128
constexpr unsigned long long EXEC_PER_PAIR = 4ull * 128 * 128 * 128;

__global__ void k_band_ranges(int64_t npiv, const uint64_t *__restrict__ ab_ptr, const uint32_t *__restrict__ ab_col,
                              const uint32_t *__restrict__ ab_np, uint32_t *__restrict__ amax,
                              uint32_t *__restrict__ bmin, uint32_t *__restrict__ bmax)
{
    __shared__ uint32_t s_am, s_bl, s_bh;
    const uint32_t I = blockIdx.x;
    if (threadIdx.x == 0) { s_am = I; s_bl = 0xffffffffu; s_bh = 0; }
    __syncthreads();
    const int64_t i = (int64_t)I * 128 + threadIdx.x;
    if (i < npiv) {
        const uint64_t s = ab_ptr[i], e = ab_ptr[i + 1];
        const uint32_t np = ab_np[i];
        atomicMax(&s_am, ab_col[s + np - 1] / 128u);
        if (e > s + np) {
            atomicMin(&s_bl, (uint32_t)((ab_col[s + np] - npiv) / 128));
            atomicMax(&s_bh, (uint32_t)((ab_col[e - 1] - npiv) / 128));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { amax[I] = s_am; bmin[I] = s_bl; bmax[I] = s_bh; }
}

// scatter the normalized pivot rows into the band tiles (warp per row)
__global__ void k_band_fill(int64_t npiv, const uint64_t *__restrict__ ab_ptr, const uint32_t *__restrict__ ab_col,
                            const uint16_t *__restrict__ ab_val, const uint64_t *__restrict__ offA,
                            const uint64_t *__restrict__ offB, const uint32_t *__restrict__ bmin,
                            uint8_t *__restrict__ tilesA, uint8_t *__restrict__ tilesB)
{
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= npiv) return;
    const uint32_t I = (uint32_t)(i / 128), k = (uint32_t)(i % 128);
    for (uint64_t q = ab_ptr[i] + lane; q < ab_ptr[i + 1]; q += 32) {
        const uint32_t c = ab_col[q];
        const uint16_t v = ab_val[q];
        uint8_t *tile;
        uint32_t o;
        if (c < (uint64_t)npiv) {
            // A tiles are written row-major (element (i, c) at toff(i, c)): the B operand of k_ahat,
            // which rewrites the off-diagonal ones as Â in the column layout toff(c, i)
            tile = tilesA + (offA[I] + (c / 128u - I)) * (uint64_t)TB;
            o = tc::toff(k, c % 128u);
        } else {
            const uint32_t nc = c - (uint32_t)npiv;
            tile = tilesB + (offB[I] + (nc / 128u - bmin[I])) * (uint64_t)TB;
            o = tc::toff(nc % 128u, k);
        }
        tile[o] = (uint8_t)(v & 0xff);
        tile[PB + o] = (uint8_t)(v >> 8);
    }
}

// padded pivots are identity rows
__global__ void k_band_pad(int64_t npiv, int64_t NB, const uint64_t *__restrict__ offA, uint8_t *__restrict__ tilesA)
{
    const int64_t i = npiv + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= NB * 128) return;
    const uint32_t I = (uint32_t)(i / 128), k = (uint32_t)(i % 128);
    tilesA[offA[I] * (uint64_t)TB + tc::toff(k, k)] = 1;
}

constexpr int DIAG_SMEM = 2 * 128 * 129 * 2;

// inv(A_JJ), unit upper triangular, as a B operand tile (K = i, MN = j)
__global__ void __launch_bounds__(128) k_diag_inv(Field F, const uint64_t *__restrict__ offA,
                                                  const uint8_t *__restrict__ tilesA, uint8_t *__restrict__ invT)
{
    extern __shared__ uint16_t dyn_inv[];
    uint16_t(*U)[129] = reinterpret_cast<uint16_t(*)[129]>(dyn_inv);
    uint16_t(*Y)[129] = reinterpret_cast<uint16_t(*)[129]>(dyn_inv + 128 * 129);
    const uint32_t J = blockIdx.x, j = threadIdx.x;
    const uint8_t *t = tilesA + offA[J] * (uint64_t)TB;     // tile (J, J) is first in row block J
    for (uint32_t idx = j; idx < 128 * 128; idx += 128) {
        const uint32_t r = idx / 128, kk = idx % 128;       // element A[kk][r] (row-major A tiles)
        const uint32_t o = tc::toff(kk, r);
        U[kk][r] = (uint16_t)(t[o] | (t[PB + o] << 8));
    }
    __syncthreads();
    for (uint32_t i = 0; i < 128; i++) Y[i][j] = (i == j) ? 1 : 0;
    for (int i = (int)j - 1; i >= 0; i--) {
        uint64_t acc = 0;
        for (uint32_t k = i + 1; k <= j; k++) acc += (uint64_t)U[i][k] * Y[k][j];
        Y[i][j] = (uint16_t)fneg(fmod64(acc, F), F);
    }
    uint8_t *o = invT + (uint64_t)J * TB;
    for (uint32_t i = 0; i < 128; i++) {
        const uint16_t v = Y[i][j];
        const uint32_t off = tc::toff(j, i);
        o[off] = (uint8_t)(v & 0xff);
        o[PB + off] = (uint8_t)(v >> 8);
    }
}

// 16 MMAs: D(HH|X|LL) (+)= A(lo,hi) x B(lo,hi), K = 128, M = N = 128
__device__ __forceinline__ void issue_mmas(uint32_t tbase, uint32_t sA, uint32_t sB, bool acc_in)
{
    const uint32_t idesc = tc::idesc_u8(128, 128);
#pragma unroll
    for (int s = 0; s < 4; s++) {
        const uint32_t off = s * 4096;
        const uint64_t dAl = tc::desc_kmajor(sA + off, 2048, 128), dAh = tc::desc_kmajor(sA + PB + off, 2048, 128);
        const uint64_t dBl = tc::desc_kmajor(sB + off, 2048, 128), dBh = tc::desc_kmajor(sB + PB + off, 2048, 128);
        const uint32_t acc = (acc_in || s > 0) ? 1u : 0u;
        // the two X products are not issued back to back (an MMA into the accumulator of the one
        // just issued waits for it)
        tc::mma_i8(tbase + 0, dAh, dBh, idesc, acc);
        tc::mma_i8(tbase + 128, dAh, dBl, idesc, acc);
        tc::mma_i8(tbase + 256, dAl, dBl, idesc, acc);
        tc::mma_i8(tbase + 128, dAl, dBh, idesc, 1u);
    }
}

// the accumulators of 16 columns reduced mod p (32-bit arithmetic, fmod_limbs)
__device__ __forceinline__ void read_R(uint32_t lane_addr, int c, uint32_t (&R)[16], const Field &F)
{
    uint32_t hh[16], xx[16], ll[16];
    __syncwarp();
    tc::tmem_ld16(lane_addr + c, hh);
    tc::tmem_ld16(lane_addr + 128 + c, xx);
    tc::tmem_ld16(lane_addr + 256 + c, ll);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; j++) R[j] = fmod_limbs(hh[j], xx[j], ll[j], F);
}

__device__ __forceinline__ void read_S(uint32_t lane_addr, int c, uint64_t (&S)[16])
{
    uint32_t hh[16], xx[16], ll[16];
    __syncwarp();
    tc::tmem_ld16(lane_addr + c, hh);
    tc::tmem_ld16(lane_addr + 128 + c, xx);
    tc::tmem_ld16(lane_addr + 256 + c, ll);
    tc::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; j++) S[j] = ((uint64_t)hh[j] << 16) + ((uint64_t)xx[j] << 8) + ll[j];
}

struct SweepArgs {
    int64_t mN, npiv, NB;
    Field F;
    const uint32_t *order, *tlead;
    const uint8_t *tilesA, *invT;
    const uint64_t *offA;
    const uint32_t *jl_ptr, *jl_idx;
    uint8_t *Xt;                   // X tiles; tile (T, J) holds C_J[T] until task (T, J) overwrites it with X_J[T]
    uint16_t *X16;
    int64_t ldX;
    const uint32_t *ab_w, *ab_np;  // op counts (Alg 2); NULL: not counted
    // back substitution (bsub_rref): X_J of target t also goes to Rout[(rrev - 1 - i) * ldR + rcol[t]]
    // for every pivot index i of block J (the reversed pivot order of the triangular solve)
    uint16_t *Rout;
    int64_t ldR, rrev;
    const uint32_t *rcol;
    unsigned long long *ops;
    int64_t prank, pworld;         // target tiles T = prank + pworld * (i0 + li) (multi-GPU row shards)
    int exp;                       // diagnostics (GBLA_SWEEP_EXP=1): no operand copies after each CTA's
                                   // first stages (the MMA loop alone; wrong results)
    int64_t i0;                    // first local tile of this batch; Xt / jmin / flags are batch-relative (li)
    // dependency-driven schedule: task q computes X_J of local tile i, (J, i) = tasks[q] (low /
    // high 32 bits).  Tasks are numbered group-major, then J-major inside a group of consecutive
    // tiles (tile_group_order), so every task waits only on tasks with smaller numbers.
    const uint64_t *tasks;         // [ntasks]
    const uint32_t *jmin;          // [nl] first block of local tile i
    uint32_t *flags;               // [nl*NB] 1 once X_J of local tile i is stored
    unsigned int *next;            // task counter
    uint32_t ntasks;
};

// first position in the ascending list v[lo, hi) with v >= key (hi if none)
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *__restrict__ v, uint32_t lo, uint32_t hi,
                                                    uint32_t key)
{
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (v[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// first block of every local target tile (NB for a tile of zero rows)
__global__ void k_tile_jmin(int64_t nl, int64_t mN, int64_t npiv, int64_t NB, int64_t prank, int64_t pworld,
                            int64_t i0, const uint32_t *__restrict__ order, const uint32_t *__restrict__ tlead,
                            uint32_t *__restrict__ jmin)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    const int64_t first = (prank + pworld * (i0 + i)) * 128;
    const uint32_t l = first < mN ? tlead[order[first]] : (uint32_t)npiv;
    jmin[i] = l >= (uint64_t)npiv ? (uint32_t)NB : l / 128u;
}

// pos[order[i]] = i (rank of every target in lead order)
__global__ void k_pos(int64_t mN, const uint32_t *__restrict__ order, uint32_t *__restrict__ pos)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < mN) pos[order[i]] = (uint32_t)i;
}

// C_J[T] into the X tiles of the batch's local tiles [i0, i1) (dense limb planes, A-operand
// layout): warp per target row
__global__ void k_cfill(int64_t mN, int64_t NB, int64_t prank, int64_t pworld, int64_t i0, int64_t i1,
                        const uint32_t *__restrict__ pos, const uint64_t *__restrict__ cd_ptr,
                        const uint32_t *__restrict__ cd_col, const uint16_t *__restrict__ cd_val,
                        const uint32_t *__restrict__ cd_np, uint8_t *__restrict__ Xt)
{
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= mN) return;
    const uint32_t ps = pos[t];
    const int64_t Tg = ps / 128;
    if (Tg < prank || (Tg - prank) % pworld != 0) return;
    const int64_t li = (Tg - prank) / pworld;
    if (li < i0 || li >= i1) return;
    const uint64_t T = (uint64_t)(li - i0), r = ps % 128;
    const uint64_t s = cd_ptr[t], e = s + cd_np[t];
    for (uint64_t q = s + lane; q < e; q += 32) {
        const uint32_t c = cd_col[q];
        const uint16_t v = cd_val[q];
        uint8_t *tile = Xt + (T * NB + c / 128) * (uint64_t)TB;
        const uint32_t o = tc::toff((uint32_t)r, c % 128);
        tile[o] = (uint8_t)(v & 0xff);
        tile[PB + o] = (uint8_t)(v >> 8);
    }
}

constexpr int NSTAGE = 3;
constexpr int PART_LD = 128;                       // running partial of long lists: u16 [128][PART_LD]
constexpr int SWEEP_SMEM = NSTAGE * 65536 + 128 * PART_LD * 2;   // 3 operand stages + the partial
constexpr int SWEEP_THREADS = 256;                 // 8 warps: two per TMEM lane quarter in the epilogue
// GBLA_SWEEP_THREADS = 128: one warp per lane quarter (each drains all 128 columns)
static int sweep_threads()
{
    const char *e = getenv("GBLA_SWEEP_THREADS");
    return e && atoi(e) == 128 ? 128 : SWEEP_THREADS;
}

// K5': persistent, dependency-driven block forward substitution.  With the band
// tiles pre-multiplied (k_ahat: Â_IJ = -A_IJ inv(A_JJ) mod p) the block step is
//   X_J = C_J inv(A_JJ) + sum_I X_I Â_IJ      (mod p)
// one accumulation of nI + 1 tile pairs and ONE epilogue.  Every CTA claims tasks
// (i, J) from a global counter in the order of a.tasks (groups of consecutive target
// tiles, J-major inside a group); the pair (C_J, inv(A_JJ)) comes first, then the X_I
// in ascending I, each waited for by its flag just before its operands are staged.
// A task only waits on tasks with smaller numbers, which were claimed earlier by
// co-resident CTAs (cooperative launch), so the schedule cannot deadlock.  Per
// 128-pivot block the chain of one target tile costs the last tile pair + one
// epilogue + the flag hand-off.  L2 reuse: the Â tiles of one J are shared by the
// tiles working on J (tile_group_size: J-major by default).
// ROLE: 0 = the sparse phase's sweep (K5'), 1 = the K14 back substitution (same code; the two
// instantiations only keep the two uses apart in profiler launch lists)
template <int ROLE>
__global__ void __launch_bounds__(SWEEP_THREADS, 1) k_sweep(SweepArgs a)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *stg = smem;
    // 8 warps: warp w drains TMEM lanes 32 (w % 4) .. +31 (= tile rows), columns 64 (w / 4) .. +63
    const int row = threadIdx.x & 127, ncol = 128 / (int)(blockDim.x >> 7), cbeg = ncol * (int)(threadIdx.x >> 7);
    uint16_t *prow = reinterpret_cast<uint16_t *>(smem + NSTAGE * 65536) + row * PART_LD;
    __shared__ uint64_t full[NSTAGE], mdone[NSTAGE], accbar;
    __shared__ uint32_t tmem_s;
    __shared__ uint32_t s_np[128], s_w[128];
    __shared__ uint32_t s_task;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_s);
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; s++) { tc::mbar_init(&full[s], 1); tc::mbar_init(&mdone[s], 1); }
        tc::mbar_init(&accbar, 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_s;
    const uint32_t lane_addr = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t ph_acc = 0;
    uint32_t ph_full = 0, ph_md = 0;           // phase bit of every stage (thread 0)
    unsigned long long opsA = 0, opsB = 0, pairs_done = 0;   // pairs_done: thread 0
    const uint32_t sStg = tc::smem_u32(stg);
    const uint32_t p = a.F.p;
    uint32_t gpair = 0;                        // stage ring position, continuous across tasks (thread 0)
    uint32_t nloads = 0;                       // diagnostics (a.exp)

    for (;;) {
        if (tid == 0) s_task = atomicAdd(a.next, 1u);
        __syncthreads();
        const uint32_t task = s_task;
        if (task >= a.ntasks) break;
        const uint64_t tv = a.tasks[task];
        const int64_t J = (uint32_t)tv, li = (uint32_t)(tv >> 32);
        const int64_t T = a.prank + a.pworld * (a.i0 + li), first = T * 128;
        const int64_t Jmin = a.jmin[li];
        const int64_t slot = first + row;
        const bool live = slot < a.mN;
        const uint32_t t = live ? a.order[slot] : 0;
        uint8_t *Xrow = a.Xt + (size_t)li * a.NB * TB;
        const uint32_t *fl = a.flags + (size_t)li * a.NB;
        const uint32_t jbase = (uint32_t)J * 128;
        if (tid < 128) {
            const uint32_t jg = jbase + tid;
            s_np[tid] = a.ab_np && jg < (uint64_t)a.npiv ? a.ab_np[jg] : 1;
            s_w[tid] = a.ab_w && jg < (uint64_t)a.npiv ? a.ab_w[jg] : 1;
        }
        const uint32_t l1 = a.jl_ptr[J + 1];
        uint32_t lb = lower_bound_u32(a.jl_idx, a.jl_ptr[J], l1, (uint32_t)Jmin);   // first I >= Jmin
        const uint32_t npair = l1 - lb + 1;            // (C_J, inv(A_JJ)), then (X_I, Â_IJ)
        pairs_done += npair;
        // the X_I already published: warp 0 reads the list's flags at once (relaxed, 32 per step) and
        // thread 0 acquires them with ONE fence (+ one proxy fence) instead of an acquire load and a
        // proxy fence per tile pair on its issue path (measured: those cost a third of the sweep)
        uint32_t nready = 0;
        if (warp == 0) {
            const uint32_t nlist = npair - 1;
            for (uint32_t b0 = 0; b0 < nlist; b0 += 32) {
                const uint32_t q = b0 + (uint32_t)lane;
                uint32_t v = 1;
                if (q < nlist) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl + a.jl_idx[lb + q]) : "memory");
                const unsigned bad = __ballot_sync(0xffffffffu, v == 0);
                if (bad) { nready = b0 + (uint32_t)__ffs(bad) - 1; break; }
                nready = b0 + 32 < nlist ? b0 + 32 : nlist;
            }
            if (lane == 0 && nready) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                fence_proxy_async_global();
            }
        }
        __syncthreads();                               // s_np / s_w are read by other threads in the epilogue
        // thread 0: the list entries (I, tile of Â_IJ) are read ahead of their use, so the global loads
        // are not on the issue path (entry e + 1's tile and entry e + 2's I while entry e is staged)
        const uint32_t nlist = npair - 1;
        uint32_t curI = 0, nxtI = 0;
        uint64_t curT = 0;
        if (tid == 0 && nlist > 0) {
            curI = __ldg(a.jl_idx + lb);
            if (nlist > 1) nxtI = __ldg(a.jl_idx + lb + 1);
            curT = __ldg(a.offA + curI) + (uint64_t)(J - curI);
        }
        // pair q into stage (gpair + q) % NSTAGE (thread 0 only, q ascending)
        auto load = [&](uint32_t q) {
            const int s = (gpair + q) % NSTAGE;
            uint8_t *sa = stg + s * 65536, *sb = sa + TB;
            if (a.exp == 1 && nloads >= (uint32_t)NSTAGE) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&full[s])) : "memory");
                return;
            }
            const bool warm = nloads >= (uint32_t)NSTAGE;
            nloads++;
            // diagnostics: 2 = skip the Â copies, 3 = skip the X copies (after the first stages)
            const bool skipB = a.exp == 2 && warm, skipA = a.exp == 3 && warm;
            tc::mbar_expect_tx(&full[s], (skipA || skipB) ? TB : 2 * TB);
            if (q == 0) {
                if (!skipB) tc::bulk_g2s(sb, a.invT + (size_t)J * TB, TB, &full[s]);
                if (!skipA) tc::bulk_g2s(sa, Xrow + (size_t)J * TB, TB, &full[s]);          // C_J (not yet overwritten)
                return;
            }
            const uint32_t I = curI;
            const uint64_t tileA = curT;
            {
                const uint32_t e = q - 1;                  // advance the read-ahead
                curI = nxtI;
                curT = e + 1 < nlist ? __ldg(a.offA + nxtI) + (uint64_t)(J - nxtI) : 0;
                nxtI = e + 2 < nlist ? __ldg(a.jl_idx + lb + e + 2) : 0;
            }
            if (!skipB) tc::bulk_g2s(sb, a.tilesA + tileA * TB, TB, &full[s]);   // Â_IJ
            if (skipA) return;
            // X_I[T] is produced by task (li, I): wait until it is published (unless the scan saw it)
            if (q - 1 >= nready) {
                if (ld_acquire(fl + I) == 0) {
                    // every CTA is resident (cooperative launch) and tasks are claimed in dependency
                    // order, so X_I is on its way; bounded all the same (never hang the GPU)
                    for (uint32_t it = 0; ld_acquire(fl + I) == 0; it++) {
                        __nanosleep(32);
                        if (it > (1u << 26)) { dev_err_latch(DEVERR_SWEEP_FLAG); break; }
                    }
                }
                fence_proxy_async_global();
            }
            tc::bulk_g2s(sa, Xrow + (size_t)I * TB, TB, &full[s]);
        };
        // exactness: one TMEM accumulation covers at most ACC_PAIRS tile pairs (K = 128 each):
        // limb sums <= 2 K 255^2 < 2^31 for K <= 16,512; longer lists (unbanded A) are folded
        // into a running partial (mod p) every ACC_PAIRS pairs
        constexpr uint32_t ACC_PAIRS = 128;
        bool have_partial = false;                     // running partial of this thread's row in prow
        if (tid == 0)
            for (uint32_t q = 0; q < npair && q < (uint32_t)NSTAGE; q++) load(q);
        for (uint32_t c0 = 0; c0 < npair; c0 += ACC_PAIRS) {
            const uint32_t c1 = c0 + ACC_PAIRS < npair ? c0 + ACC_PAIRS : npair;
            if (tid == 0) {
                for (uint32_t q = c0; q < c1; q++) {
                    const int s = (gpair + q) % NSTAGE;
                    tc::mbar_wait(&full[s], (ph_full >> s) & 1u);
                    ph_full ^= 1u << s;
                    tc::fence_after();
                    issue_mmas(tbase, sStg + s * 65536, sStg + s * 65536 + TB, q > c0);
                    if (q + NSTAGE < npair) tc::commit(&mdone[s]);     // stage s is reloaded for q + NSTAGE
                    // refill the stage of the previous pair once its MMAs are done
                    if (q >= 1 && q - 1 + NSTAGE < npair) {
                        const int sp = (gpair + q - 1) % NSTAGE;
                        tc::mbar_wait(&mdone[sp], (ph_md >> sp) & 1u);
                        ph_md ^= 1u << sp;
                        load(q - 1 + NSTAGE);
                    }
                }
                tc::commit(&accbar);
            }
            tc::mbar_wait(&accbar, ph_acc);
            ph_acc ^= 1;
            tc::fence_after();
            if (c1 < npair) {                          // fold this chunk into the partial, free TMEM
#pragma unroll 1
                for (int c = cbeg; c < cbeg + ncol; c += 16) {
                    uint32_t Rv[16];
                    read_R(lane_addr, c, Rv, a.F);
#pragma unroll
                    for (int j = 0; j < 16; j++) {
                        uint32_t v = Rv[j];
                        if (have_partial) {
                            v += prow[c + j];
                            v = v >= p ? v - p : v;
                        }
                        prow[c + j] = (uint16_t)v;
                    }
                }
                have_partial = true;
                tc::fence_before();
                __syncthreads();
                tc::fence_after();
            }
        }
        if (tid == 0) gpair = (gpair + npair) % NSTAGE;
        // epilogue: X_J = S (+ partial) mod p -> limb-plane tile (global) [+ C' u16], op counts (Alg 2)
        uint8_t *xt = Xrow + (size_t)J * TB;
#pragma unroll 1
        for (int c8 = cbeg; c8 < cbeg + ncol; c8 += 16) {
            const int c = c8 / 16;
            uint32_t Rv[16];
            read_R(lane_addr, c8, Rv, a.F);
            uint8_t lo8[16], hi8[16];
            uint16_t xs[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                uint32_t x = Rv[j];
                if (have_partial) {
                    x += prow[c8 + j];
                    x = x >= p ? x - p : x;
                }
                lo8[j] = (uint8_t)(x & 0xff);
                hi8[j] = (uint8_t)(x >> 8);
                xs[j] = (uint16_t)x;
                if (x && live) {
                    opsA += s_np[c * 16 + j] - 1;
                    opsB += s_w[c * 16 + j] - s_np[c * 16 + j];
                }
            }
            const uint32_t o = tc::toff(row, c * 16);
            *reinterpret_cast<uint4 *>(xt + o) = *reinterpret_cast<uint4 *>(lo8);
            *reinterpret_cast<uint4 *>(xt + PB + o) = *reinterpret_cast<uint4 *>(hi8);
            if (a.X16 && live) {
#pragma unroll
                for (int j = 0; j < 16; j++)
                    if (jbase + c * 16 + j < (uint64_t)a.npiv) a.X16[(size_t)t * a.ldX + jbase + c * 16 + j] = xs[j];
            }
            if (a.Rout && live) {
                uint16_t *rc = a.Rout + a.rcol[t];
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const int64_t i = (int64_t)jbase + c * 16 + j;
                    if (i < a.npiv) rc[(size_t)(a.rrev - 1 - i) * a.ldR] = xs[j];
                }
            }
        }
        fence_proxy_async_global();     // X_J is read by later tasks through the async proxy
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        if (tid == 0) {
            __threadfence();
            st_release(a.flags + (size_t)li * a.NB + J, 1u);
        }
    }
    for (int o = 16; o; o >>= 1) {
        opsA += __shfl_xor_sync(0xffffffffu, opsA, o);
        opsB += __shfl_xor_sync(0xffffffffu, opsB, o);
    }
    if ((tid & 31) == 0) {
        atomicAdd(&a.ops[0], opsA);
        atomicAdd(&a.ops[1], opsB);
    }
    if (tid == 0) atomicAdd(&a.ops[2], pairs_done);
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

// Â_IJ = -A_IJ inv(A_JJ) mod p for every off-diagonal band tile, in place: A_IJ arrives
// row-major (element (i, k) at toff(i, k), k_band_fill) and leaves as Â in the layout the sweep
// uses (element (i, j) at toff(j, i)).  As a tcgen05 product D[j][i] = sum_k W[k][j] A_IJ[i][k]:
// the stored inv(A_JJ) tile is the A operand as is (toff(j, k) holds W[k][j]) and the row-major
// A_IJ tile is the B operand as is (toff(i, k) holds A_IJ[i][k]).  The epilogue thread j writes
// its 128 values at toff(j, i), negated.  One CTA per tile.
__global__ void __launch_bounds__(128, 1) k_ahat(Field F, int64_t NB, const uint64_t *__restrict__ offA,
                                                 const uint32_t *__restrict__ amax, const uint64_t *__restrict__ tile_I,
                                                 int64_t ntile, uint8_t *__restrict__ tilesA,
                                                 const uint8_t *__restrict__ invT)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *sW = smem, *sB = smem + TB;                // W (A operand), A_IJ (B operand)
    __shared__ uint64_t bar, accbar;
    __shared__ uint32_t tmem_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_s);
    if (tid == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&accbar, 1); }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_s, lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
    uint32_t ph = 0, pha = 0;
    for (int64_t q = blockIdx.x; q < ntile; q += gridDim.x) {
        const uint64_t code = tile_I[q];
        const uint32_t I = (uint32_t)(code >> 32), J = (uint32_t)code;
        uint8_t *tA = tilesA + (offA[I] + (uint64_t)(J - I)) * TB;
        if (tid == 0) {
            tc::mbar_expect_tx(&bar, 2 * TB);
            tc::bulk_g2s(sW, invT + (size_t)J * TB, TB, &bar);
            tc::bulk_g2s(sB, tA, TB, &bar);
        }
        tc::mbar_wait(&bar, ph);
        ph ^= 1;
        tc::fence_after();
        if (tid == 0) {
            issue_mmas(tbase, tc::smem_u32(sW), tc::smem_u32(sB), false);
            tc::commit(&accbar);
        }
        tc::mbar_wait(&accbar, pha);
        pha ^= 1;
        tc::fence_after();
#pragma unroll 1
        for (int c = 0; c < 128; c += 16) {
            uint32_t Rv[16];
            read_R(lane_addr, c, Rv, F);
            uint8_t lo8[16], hi8[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t v = Rv[j] ? F.p - Rv[j] : 0;
                lo8[j] = (uint8_t)(v & 0xff);
                hi8[j] = (uint8_t)(v >> 8);
            }
            const uint32_t o = tc::toff(tid, c);          // thread = j, columns c.. = i
            *reinterpret_cast<uint4 *>(tA + o) = *reinterpret_cast<uint4 *>(lo8);
            *reinterpret_cast<uint4 *>(tA + PB + o) = *reinterpret_cast<uint4 *>(hi8);
        }
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
    }
    if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

struct UpdArgs {
    int64_t mN, npiv, nN, NB;
    Field F;
    const uint32_t *order, *tlead;
    const uint8_t *Xt, *tilesB;
    const uint64_t *offB;
    const uint32_t *bmin, *kl_ptr, *kl_idx;
    uint16_t *D;
    int64_t ldD;
    int64_t prank, pworld;         // target tiles T = prank + pworld * (i0 + blockIdx.y)
    int64_t i0;                    // first local tile of the batch (Xt is batch-relative)
};

constexpr int UPD_NS = 3;                        // operand stages (one CTA per SM either way)
constexpr int UPD_SMEM = UPD_NS * 65536;

__global__ void __launch_bounds__(128, 1) k_update_tc(UpdArgs a)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[UPD_NS], mdone[UPD_NS], accbar;
    __shared__ uint32_t tmem_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t K = blockIdx.x, T = a.prank + a.pworld * (a.i0 + (int64_t)blockIdx.y), first = T * 128;
    const uint32_t lead0 = a.tlead[a.order[first]];
    if (lead0 >= (uint64_t)a.npiv) return;
    const int64_t Jmin = lead0 / 128;
    const uint32_t l1 = a.kl_ptr[K + 1];
    const uint32_t lb = lower_bound_u32(a.kl_idx, a.kl_ptr[K], l1, (uint32_t)Jmin);
    const uint32_t nI = l1 - lb;
    if (nI == 0) return;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_s);
    if (tid == 0) {
        for (int q = 0; q < UPD_NS; q++) { tc::mbar_init(&full[q], 1); tc::mbar_init(&mdone[q], 1); }
        tc::mbar_init(&accbar, 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_s;
    const uint32_t sStg = tc::smem_u32(smem);
    const uint8_t *Xrow = a.Xt + (size_t)blockIdx.y * a.NB * TB;
    uint32_t ph_full = 0, ph_md = 0, ph_acc = 0;       // phase bit of every stage (thread 0) / all
    // thread 0: list entries read ahead of their use (entry it + 1's tile and entry it + 2's I while
    // entry it is staged), so no dependent global load sits on the issue path
    uint32_t curI = 0, nxtI = 0;
    uint64_t curT = 0;
    if (tid == 0) {
        curI = __ldg(a.kl_idx + lb);
        if (nI > 1) nxtI = __ldg(a.kl_idx + lb + 1);
        curT = __ldg(a.offB + curI) + (uint64_t)(K - __ldg(a.bmin + curI));
    }
    auto load = [&](uint32_t it) {                     // thread 0 only, it ascending
        const uint32_t I = curI;
        const uint64_t tileB = curT;
        curI = nxtI;
        curT = it + 1 < nI ? __ldg(a.offB + nxtI) + (uint64_t)(K - __ldg(a.bmin + nxtI)) : 0;
        nxtI = it + 2 < nI ? __ldg(a.kl_idx + lb + it + 2) : 0;
        const int s = it % UPD_NS;
        tc::mbar_expect_tx(&full[s], 2 * TB);
        tc::bulk_g2s(smem + s * 65536, Xrow + (size_t)I * TB, TB, &full[s]);
        tc::bulk_g2s(smem + s * 65536 + TB, a.tilesB + tileB * TB, TB, &full[s]);
    };
    if (tid == 0)
        for (uint32_t q = 0; q < nI && q < (uint32_t)UPD_NS; q++) load(q);
    const int64_t slot = first + tid;
    const bool live = slot < a.mN;
    uint16_t *drow = live ? a.D + (size_t)a.order[slot] * a.ldD + K * 128 : nullptr;
    const uint32_t lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
    const uint32_t p = a.F.p;
    // one TMEM accumulation covers at most 128 tile pairs (K <= 16,384: exact s32 limb sums);
    // longer lists (unbanded B) subtract each chunk from D
    constexpr uint32_t ACC_PAIRS = 128;
    for (uint32_t c0 = 0; c0 < nI; c0 += ACC_PAIRS) {
        const uint32_t c1 = c0 + ACC_PAIRS < nI ? c0 + ACC_PAIRS : nI;
        if (tid == 0) {
            for (uint32_t it = c0; it < c1; it++) {
                const int s = it % UPD_NS;
                tc::mbar_wait(&full[s], (ph_full >> s) & 1u);
                ph_full ^= 1u << s;
                tc::fence_after();
                issue_mmas(tbase, sStg + s * 65536, sStg + s * 65536 + TB, it > c0);
                if (it + UPD_NS < nI) tc::commit(&mdone[s]);       // stage s is reloaded for it + UPD_NS
                // refill the stage of the previous pair once its MMAs are done (this pair's MMAs
                // are queued behind them: the tensor pipe never waits for the refill)
                if (it >= 1 && it - 1 + UPD_NS < nI) {
                    const int sp = (it - 1) % UPD_NS;
                    tc::mbar_wait(&mdone[sp], (ph_md >> sp) & 1u);
                    ph_md ^= 1u << sp;
                    load(it - 1 + UPD_NS);
                }
            }
            tc::commit(&accbar);
        }
        // this thread's D row segment (256 B) read while the MMAs run: the epilogue's global loads
        // are off the path after the accumulator is done
        uint4 dv[16];
        if (live) {
#pragma unroll
            for (int j = 0; j < 16; j++) dv[j] = *reinterpret_cast<const uint4 *>(drow + 8 * j);
        }
        tc::mbar_wait(&accbar, ph_acc);
        ph_acc ^= 1;
        tc::fence_after();
#pragma unroll
        for (int c = 0; c < 128; c += 16) {
            uint32_t Rv[16];
            read_R(lane_addr, c, Rv, a.F);
            if (!live) continue;
            uint4 v[2];
            v[0] = dv[c / 8];
            v[1] = dv[c / 8 + 1];
            uint16_t *d = reinterpret_cast<uint16_t *>(v);
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const uint32_t s = Rv[j];
                const uint32_t x = d[j];
                d[j] = (uint16_t)(x >= s ? x - s : x + p - s);
            }
            *reinterpret_cast<uint4 *>(drow + c) = v[0];
            *reinterpret_cast<uint4 *>(drow + c + 8) = v[1];
        }
        tc::fence_before();
        __syncthreads();                               // accumulator free for the next chunk
        tc::fence_after();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

}  // namespace

void band_free(gbla_mat h)
{
    delete h->bt;
    h->bt = nullptr;
}


static gbla_status band_build(gbla_mat h)
{
    if (h->bt) return GBLA_OK;
    cudaStream_t st = h->stream;
    BandTiles *bt = new BandTiles();
    h->bt = bt;
    const int64_t npiv = h->npiv, nN = h->nN;
    bt->NB = (npiv + 127) / 128;
    bt->NNB = (nN + 127) / 128;
    bt->ntiles = (h->mN + 127) / 128;
    const int64_t NB = bt->NB, NNB = bt->NNB;
    GBLA_TRY(dalloc_t(h, 3, &bt->ops));
    GBLA_CUDA_TRY(cudaMemsetAsync(bt->ops, 0, 24, st));
    if (NB == 0) return GBLA_OK;
    GBLA_TRY(dalloc_t(h, NB, &bt->amax));
    GBLA_TRY(dalloc_t(h, NB, &bt->bmin));
    GBLA_TRY(dalloc_t(h, NB, &bt->bmax));
    k_band_ranges<<<(unsigned)NB, 128, 0, st>>>(npiv, h->ab_ptr, h->ab_col, h->ab_np, bt->amax, bt->bmin, bt->bmax);
    note_launch();
    std::vector<uint32_t> amax(NB), bmin(NB), bmax(NB);
    GBLA_CUDA_TRY(cudaMemcpyAsync(amax.data(), bt->amax, NB * 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bmin.data(), bt->bmin, NB * 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bmax.data(), bt->bmax, NB * 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<uint64_t> offA(NB), offB(NB);
    std::vector<std::vector<uint32_t>> jl(NB), kl(NNB > 0 ? NNB : 1);
    uint64_t nA = 0, nB = 0;
    for (int64_t I = 0; I < NB; I++) {
        if (amax[I] >= NB) amax[I] = NB - 1;
        offA[I] = nA;
        nA += amax[I] - I + 1;
        for (uint32_t J = I + 1; J <= amax[I]; J++)
            jl[J].push_back((uint32_t)I);
        offB[I] = nB;
        if (bmin[I] <= bmax[I] && bmin[I] != 0xffffffffu) {
            nB += bmax[I] - bmin[I] + 1;
            for (uint32_t K = bmin[I]; K <= bmax[I]; K++) kl[K].push_back((uint32_t)I);
        }
    }
    bt->nA = nA;
    bt->nB = nB;
    std::vector<uint32_t> jptr(NB + 1), kptr(NNB + 1), jidx, kidx;
    for (int64_t J = 0; J < NB; J++) { jptr[J] = (uint32_t)jidx.size(); jidx.insert(jidx.end(), jl[J].begin(), jl[J].end()); }
    jptr[NB] = (uint32_t)jidx.size();
    for (int64_t K = 0; K < NNB; K++) { kptr[K] = (uint32_t)kidx.size(); kidx.insert(kidx.end(), kl[K].begin(), kl[K].end()); }
    kptr[NNB] = (uint32_t)kidx.size();
    GBLA_TRY(dalloc_t(h, NB, &bt->offA));
    GBLA_TRY(dalloc_t(h, NB, &bt->offB));
    GBLA_TRY(dalloc_t(h, NB + 1, &bt->jl_ptr));
    GBLA_TRY(dalloc_t(h, jidx.size() + 1, &bt->jl_idx));
    GBLA_TRY(dalloc_t(h, NNB + 1, &bt->kl_ptr));
    GBLA_TRY(dalloc_t(h, kidx.size() + 1, &bt->kl_idx));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bt->amax, amax.data(), NB * 4, cudaMemcpyHostToDevice, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bt->offA, offA.data(), NB * 8, cudaMemcpyHostToDevice, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bt->offB, offB.data(), NB * 8, cudaMemcpyHostToDevice, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bt->jl_ptr, jptr.data(), (NB + 1) * 4, cudaMemcpyHostToDevice, st));
    if (!jidx.empty())
        GBLA_CUDA_TRY(cudaMemcpyAsync(bt->jl_idx, jidx.data(), jidx.size() * 4, cudaMemcpyHostToDevice, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(bt->kl_ptr, kptr.data(), (NNB + 1) * 4, cudaMemcpyHostToDevice, st));
    if (!kidx.empty())
        GBLA_CUDA_TRY(cudaMemcpyAsync(bt->kl_idx, kidx.data(), kidx.size() * 4, cudaMemcpyHostToDevice, st));
    GBLA_TRY(dalloc(h, nA * TB + 16, (void **)&bt->tilesA));
    GBLA_TRY(dalloc(h, (nB > 0 ? nB : 1) * TB + 16, (void **)&bt->tilesB));
    GBLA_TRY(dalloc(h, NB * TB + 16, (void **)&bt->invT));
    GBLA_CUDA_TRY(cudaMemsetAsync(bt->tilesA, 0, nA * TB, st));
    if (nB) GBLA_CUDA_TRY(cudaMemsetAsync(bt->tilesB, 0, nB * TB, st));
    k_band_fill<<<grid_for(npiv * 32, 256), 256, 0, st>>>(npiv, h->ab_ptr, h->ab_col, h->ab_val, bt->offA, bt->offB,
                                                          bt->bmin, bt->tilesA, bt->tilesB);
    if (NB * 128 > npiv) k_band_pad<<<1, 128, 0, st>>>(npiv, NB, bt->offA, bt->tilesA);
    {
        static unsigned long long attr = 0;   // devices done (dev_bit)
        if (!(attr & dev_bit())) {
            GBLA_CUDA_TRY(cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, DIAG_SMEM));
            attr |= dev_bit();
        }
    }
    k_diag_inv<<<(unsigned)NB, 128, DIAG_SMEM, st>>>(h->F, bt->offA, bt->tilesA, bt->invT);
    note_launch(3);
    GBLA_CUDA_TRY(cudaGetLastError());
    // Â_IJ = -A_IJ inv(A_JJ) for every off-diagonal band tile (the sweep's B operands)
    {
        std::vector<uint64_t> tl;
        for (int64_t I = 0; I < NB; I++)
            for (uint32_t J = (uint32_t)I + 1; J <= amax[I]; J++) tl.push_back(((uint64_t)I << 32) | J);
        if (!tl.empty()) {
            uint64_t *dtl;
            GBLA_TRY(dalloc_t(h, tl.size(), &dtl));
            GBLA_CUDA_TRY(cudaMemcpyAsync(dtl, tl.data(), tl.size() * 8, cudaMemcpyHostToDevice, st));
            static unsigned long long attr2 = 0;   // devices done (dev_bit)
            if (!(attr2 & dev_bit())) {
                GBLA_CUDA_TRY(cudaFuncSetAttribute(k_ahat, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TB));
                attr2 |= dev_bit();
            }
            const int64_t nt = (int64_t)tl.size();
            const int64_t grid = nt < 2 * (int64_t)h->ctx->sm_count ? nt : 2 * (int64_t)h->ctx->sm_count;
            k_ahat<<<(unsigned)grid, 128, 2 * TB, st>>>(h->F, NB, bt->offA, bt->amax, dtl, nt, bt->tilesA, bt->invT);
            note_launch();
            GBLA_CUDA_TRY(cudaGetLastError());
            // the host list must outlive the async copy
            GBLA_CUDA_TRY(cudaStreamSynchronize(st));
        }
    }
    return GBLA_OK;
}

// ---- host side -------------------------------------------------------------
static inline int64_t local_tiles(int64_t ntiles, int prank, int pworld)
{
    return ntiles > prank ? (ntiles - prank + pworld - 1) / pworld : 0;
}

// X tiles per batch of target tiles: all of them if they fit beside what is
// already allocated (keeping a reserve for the echelon), else as many as fit
// (1172 tiles x 6641 blocks x 32 KB would be 255 GB).
static int64_t xt_batch_tiles(gbla_mat h, int64_t nl)
{
    const int64_t per_tile = h->bt->NB * (int64_t)TB;
    const char *e = getenv("GBLA_XT_BATCH");          // tests: force small batches
    if (e && atoll(e) > 0) return atoll(e) < nl ? atoll(e) : nl;
    if (nl * per_tile <= ((int64_t)8 << 30)) return nl;   // small: no need to ask the driver
    size_t fr = 0, tot = 0;
    const int64_t reserve = (int64_t)4 << 30;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) { cudaGetLastError(); return nl; }
    if ((int64_t)fr - reserve >= nl * per_tile) return nl;         // fits in what the driver has free
    if (h->ctx->memq) fr = h->ctx->memq(h->ctx->memq_user);      // the caller's allocator (torch: + cached)
    int64_t budget = (int64_t)fr - reserve;
    if (budget < per_tile) budget = per_tile;
    const int64_t b = budget / per_tile;
    return b < nl ? (b > 0 ? b : 1) : nl;
}

// Target tiles per task group of the sweep (GBLA_SWEEP_GROUP / GBLA_BSUB_GROUP = n; default: one
// group, i.e. plain J-major order).  Small groups keep a target tile's X_I in L2 between its
// consecutive J (several J of one tile in flight) and large ones share each Â tile among many
// tiles; measured on c2 (sparse sweep / back substitution): groups of 4 and 8 tiles are chain-bound
// (368 / 190 ms against 107 ms J-major: a tile's chain advances one J per last pair + epilogue +
// flag hand-off, slower than 18-37 CTAs consume its tasks), 32 and 64 equal to J-major.
static int64_t tile_group_size(int64_t grid, double pairs, int64_t nl, const char *env)
{
    (void)grid;
    (void)pairs;
    const char *e = getenv(env);
    int64_t g = e && atoll(e) > 0 ? atoll(e) : nl;
    if (g < 1) g = 1;
    return g < nl ? g : (nl > 0 ? nl : 1);
}

// What one sweep solves: x_t A = c_t for the targets t (A = the band tiles of bt, C in bt->Xt)
struct SweepSrc {
    BandTiles *bt;
    int64_t mN, npiv;                        // targets, pivots (A is npiv x npiv)
    const uint32_t *order, *tlead;           // targets sorted by lead; sigma(lead) per target
    uint16_t *X16 = nullptr;                 // optional u16 copy of X (row t, ldX)
    int64_t ldX = 0;
    const uint32_t *ab_w = nullptr, *ab_np = nullptr;   // Alg 2 op counts (NULL: none)
    uint16_t *Rout = nullptr;                // optional reversed transposed output (bsub_rref)
    int64_t ldR = 0, rrev = 0;
    const uint32_t *rcol = nullptr;
    int kt = KT_SWEEP;                       // timer family (-1: none)
    const char *group_env = "GBLA_SWEEP_GROUP";   // tile_group_size override
};

static gbla_status sweep_run(gbla_mat h, const SweepSrc &src, int prank, int pworld, int64_t i0, int64_t i1);

// K5' for the local target tiles [i0, i1) (T = prank + pworld * i)
static gbla_status tc_sweep_batch(gbla_mat h, int prank, int pworld, int64_t i0, int64_t i1, bool want_x16)
{
    SweepSrc src;
    src.bt = h->bt; src.mN = h->mN; src.npiv = h->npiv; src.order = h->order; src.tlead = h->tlead;
    src.X16 = want_x16 ? h->X : nullptr; src.ldX = h->ldX;
    src.ab_w = h->ab_w; src.ab_np = h->ab_np;
    return sweep_run(h, src, prank, pworld, i0, i1);
}

static gbla_status sweep_run(gbla_mat h, const SweepSrc &src, int prank, int pworld, int64_t i0, int64_t i1)
{
    cudaStream_t st = h->stream;
    BandTiles *bt = src.bt;
    const int64_t nl = i1 - i0;
    const int64_t NB = bt->NB;
    if (NB == 0 || nl <= 0) return GBLA_OK;
    // set on the current device every time (one context per device; the call is cheap)
    const void *kfn = src.Rout ? (const void *)k_sweep<1> : (const void *)k_sweep<0>;
    GBLA_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SWEEP_SMEM));
    int occ = 0;
    GBLA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, sweep_threads(), SWEEP_SMEM));
    if (occ < 1) { set_error("k_sweep does not fit on an SM"); return GBLA_E_INTERNAL; }
    // task schedule: first block of every local tile -> grouped task list
    uint32_t *jmin, *flags;
    uint64_t *tasks;
    unsigned int *next;
    GBLA_TRY(dalloc_t(h, nl, &jmin));
    GBLA_TRY(dalloc_t(h, (size_t)nl * NB, &flags));
    GBLA_TRY(dalloc_t(h, 1, &next));
    k_tile_jmin<<<grid_for(nl, 256), 256, 0, st>>>(nl, src.mN, src.npiv, NB, prank, pworld, i0, src.order, src.tlead,
                                                     jmin);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    std::vector<uint32_t> hj(nl), hjl(NB + 1);
    GBLA_CUDA_TRY(cudaMemcpyAsync(hj.data(), jmin, nl * 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(hjl.data(), bt->jl_ptr, (NB + 1) * 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)nl * NB * 4, st));
    GBLA_CUDA_TRY(cudaMemsetAsync(next, 0, 4, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    for (int64_t q = 1; q < nl; q++)
        if (hj[q] < hj[q - 1]) { set_error("k_sweep: target tiles not sorted by lead"); return GBLA_E_INTERNAL; }
    int64_t grid = (int64_t)h->ctx->sm_count * occ;
    std::vector<uint64_t> ht;
    {
        // mean tile pairs per task (band depth) over the active blocks
        double pairs = 0.0, nact = 0.0;
        for (int64_t J = (nl ? hj[0] : NB); J < NB; J++) { pairs += hjl[J + 1] - hjl[J] + 1.0; nact += 1.0; }
        const int64_t GT = tile_group_size(grid, nact > 0 ? pairs / nact : 1.0, nl, src.group_env);
        // group-major, then J-major over the group's tiles active at J (a prefix: sorted by lead)
        for (int64_t g0 = 0; g0 < nl; g0 += GT) {
            const int64_t g1 = g0 + GT < nl ? g0 + GT : nl;
            int64_t i = g0;
            for (int64_t J = hj[g0]; J < NB; J++) {
                while (i < g1 && hj[i] <= (uint64_t)J) i++;
                for (int64_t q = g0; q < i; q++) ht.push_back(((uint64_t)q << 32) | (uint64_t)J);
            }
        }
        if (ht.size() >= 0xffffffffull) { set_error("k_sweep: too many tasks"); return GBLA_E_INTERNAL; }
    }
    const uint32_t ntasks = (uint32_t)ht.size();
    if (ntasks == 0) return GBLA_OK;
    GBLA_TRY(dalloc_t(h, ht.size(), &tasks));
    GBLA_CUDA_TRY(cudaMemcpyAsync(tasks, ht.data(), ht.size() * 8, cudaMemcpyHostToDevice, st));
    // (pageable source: the copy is staged before cudaMemcpyAsync returns)
    SweepArgs a;
    a.mN = src.mN; a.npiv = src.npiv; a.NB = NB; a.F = h->F;
    a.order = src.order; a.tlead = src.tlead;
    a.tilesA = bt->tilesA; a.invT = bt->invT; a.offA = bt->offA;
    a.jl_ptr = bt->jl_ptr; a.jl_idx = bt->jl_idx;
    a.Xt = bt->Xt; a.X16 = src.X16; a.ldX = src.ldX;
    a.ab_w = src.ab_w; a.ab_np = src.ab_np; a.ops = bt->ops;
    a.Rout = src.Rout; a.ldR = src.ldR; a.rrev = src.rrev; a.rcol = src.rcol;
    a.prank = prank; a.pworld = pworld; a.i0 = i0;
    a.tasks = tasks; a.jmin = jmin; a.flags = flags; a.next = next; a.ntasks = ntasks;
    a.exp = getenv("GBLA_SWEEP_EXP") ? atoi(getenv("GBLA_SWEEP_EXP")) : 0;
    if (grid > (int64_t)ntasks) grid = ntasks;
    // co-residency of every CTA is what makes the flag waits safe: cooperative launch
    void *kargs[] = {&a};
    if (src.kt >= 0) kt_mark(h, src.kt);
    GBLA_CUDA_TRY(cudaLaunchCooperativeKernel(kfn, dim3((unsigned)grid), dim3(sweep_threads()), kargs,
                                              (size_t)SWEEP_SMEM, st));
    if (src.kt >= 0) kt_mark(h, src.kt);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

// K7' for the local target tiles [i0, i1)
static gbla_status tc_update_batch(gbla_mat h, int prank, int pworld, int64_t i0, int64_t i1)
{
    cudaStream_t st = h->stream;
    BandTiles *bt = h->bt;
    const int64_t nl = i1 - i0;
    if (bt->NB == 0 || bt->NNB == 0 || nl <= 0) return GBLA_OK;
    static unsigned long long attr = 0;   // devices done (dev_bit)
    if (!(attr & dev_bit())) {
        GBLA_CUDA_TRY(cudaFuncSetAttribute(k_update_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, UPD_SMEM));
        attr |= dev_bit();
    }
    UpdArgs a;
    a.mN = h->mN; a.npiv = h->npiv; a.nN = h->nN; a.NB = bt->NB; a.F = h->F;
    a.order = h->order; a.tlead = h->tlead;
    a.Xt = bt->Xt; a.tilesB = bt->tilesB; a.offB = bt->offB; a.bmin = bt->bmin;
    a.kl_ptr = bt->kl_ptr; a.kl_idx = bt->kl_idx; a.D = h->D; a.ldD = h->ldD;
    a.prank = prank; a.pworld = pworld; a.i0 = i0;
    for (int64_t y0 = 0; y0 < nl; y0 += 65535) {       // gridDim.y <= 65535
        const int64_t ny = nl - y0 < 65535 ? nl - y0 : 65535;
        a.i0 = i0 + y0;
        UpdArgs b = a;
        b.Xt = bt->Xt + (size_t)y0 * bt->NB * TB;
        kt_mark(h, KT_UPDATE);
        k_update_tc<<<dim3((unsigned)bt->NNB, (unsigned)ny), 128, UPD_SMEM, st>>>(b);
        kt_mark(h, KT_UPDATE);
        note_launch();
    }
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

// the Alg 2 modMAC counts accumulated by the sweeps so far: [A part, B part]
gbla_status tc_read_ops(gbla_mat h, unsigned long long ops[2])
{
    ops[0] = ops[1] = 0;
    if (!h->bt) return GBLA_OK;
    unsigned long long o3[3];
    GBLA_CUDA_TRY(cudaMemcpyAsync(o3, h->bt->ops, 24, cudaMemcpyDeviceToHost, h->stream));
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    ops[0] = o3[0];
    ops[1] = o3[1];
    h->kexec[KT_SWEEP] = o3[2] * EXEC_PER_PAIR;
    return GBLA_OK;
}

// The sparse phase of the local target tiles of rank prank of pworld: in batches of
// target tiles (X tiles = C_J, then X_J), sweep (C' = C A^-1) and, if `update`,
// D -= C' B.  Without `update` every X tile must stay resident for a later
// gbla_update_D (one batch).  After a fused pass the band and X tiles are released.
static gbla_status tc_sparse(gbla_mat h, int prank, int pworld, bool want_x16, bool update)
{
    cudaStream_t st = h->stream;
    GBLA_TRY(band_build(h));
    BandTiles *bt = h->bt;
    const int64_t NB = bt->NB;
    const int64_t nl = local_tiles(bt->ntiles, prank, pworld);
    if (NB == 0 || nl == 0) return GBLA_OK;
    if (!bt->tilesA) { set_error("sparse phase: band tiles already released"); return GBLA_E_ORDER; }
    if (!bt->Xt) {
        bt->xt_cap = update ? xt_batch_tiles(h, nl) : nl;
        GBLA_TRY(dalloc(h, (size_t)bt->xt_cap * NB * TB + 16, (void **)&bt->Xt));
    }
    const int64_t per = bt->xt_cap < nl ? bt->xt_cap : nl;
    if (!update && per < nl) { set_error("unfused reduce_C needs every C' tile resident"); return GBLA_E_NOMEM; }
    uint32_t *pos;
    GBLA_TRY(dalloc_t(h, h->mN, &pos));
    k_pos<<<grid_for(h->mN, 256), 256, 0, st>>>(h->mN, h->order, pos);
    note_launch();
    for (int64_t i0 = 0; i0 < nl; i0 += per) {
        const int64_t i1 = i0 + per < nl ? i0 + per : nl;
        GBLA_CUDA_TRY(cudaMemsetAsync(bt->Xt, 0, (size_t)(i1 - i0) * NB * TB, st));
        k_cfill<<<grid_for(h->mN * 32, 256), 256, 0, st>>>(h->mN, NB, prank, pworld, i0, i1, pos, h->cd_ptr,
                                                           h->cd_col, h->cd_val, h->cd_np, bt->Xt);
        note_launch();
        GBLA_CUDA_TRY(cudaGetLastError());
        GBLA_TRY(tc_sweep_batch(h, prank, pworld, i0, i1, want_x16));
        if (update) GBLA_TRY(tc_update_batch(h, prank, pworld, i0, i1));
    }
    return GBLA_OK;
}

// device buffers of the band / X tiles are dead after the update: give them back
// before the echelon (c4 needs the memory)
void band_release(gbla_mat h)
{
    BandTiles *bt = h->bt;
    if (!bt) return;
    dfree(h, bt->tilesA); bt->tilesA = nullptr;
    dfree(h, bt->tilesB); bt->tilesB = nullptr;
    dfree(h, bt->invT); bt->invT = nullptr;
    dfree(h, bt->Xt); bt->Xt = nullptr;
    bt->xt_cap = 0;
}

// C' = C A^-1 on the whole C (single GPU; gbla_reduce_C); fused: also D -= C' B
gbla_status reduce_c_tc(gbla_mat h, bool want_x16, bool fused)
{
    if (want_x16) GBLA_TRY(ensure_x(h));
    if (h->mN == 0 || h->npiv == 0) {     // C is empty: C' = 0, D_new = D
        h->have_xt = true;
        return GBLA_OK;
    }
    GBLA_TRY(tc_sparse(h, 0, 1, want_x16, fused));
    if (h->bt) h->bt->swept = true;
    if (fused) band_release(h);
    unsigned long long ops[2];
    GBLA_TRY(tc_read_ops(h, ops));
    GBLA_TRY(sweep_dev_err(h->stream, "gbla_reduce_C"));
    h->sparse_ops += ops[0] + (fused ? ops[1] : 0);
    h->kwork[KT_SWEEP] = ops[0];
    if (fused) h->kwork[KT_UPDATE] = ops[1];
    h->have_xt = !fused;
    return GBLA_OK;
}

// D <- D - C' B with the C' tiles of an unfused reduce_c_tc (single GPU; gbla_update_D)
gbla_status update_d_tc(gbla_mat h)
{
    if (h->mN == 0 || h->npiv == 0) return GBLA_OK;
    if (!h->bt || !h->bt->swept || !h->bt->Xt) { set_error("update_d_tc: no C' tiles"); return GBLA_E_INTERNAL; }
    GBLA_TRY(tc_update_batch(h, 0, 1, 0, local_tiles(h->bt->ntiles, 0, 1)));
    unsigned long long ops[2];
    GBLA_TRY(tc_read_ops(h, ops));
    h->sparse_ops += ops[1];
    h->kwork[KT_UPDATE] = ops[1];
    band_release(h);
    return GBLA_OK;
}

// multi-GPU / emulated ranks: the sparse phase of one row shard (fused)
gbla_status tc_shard(gbla_mat h, int prank, int pworld)
{
    if (h->mN == 0 || h->npiv == 0) return GBLA_OK;
    return tc_sparse(h, prank, pworld, false, true);
}
int64_t tc_ntiles(gbla_mat h) { return h->bt ? h->bt->ntiles : (h->mN + 127) / 128; }
unsigned long long *tc_ops_dev(gbla_mat h) { return h->bt ? h->bt->ops : nullptr; }

// ---- K14: the fully reduced echelon from a row echelon form (back substitution) -------------
//
// R13 asks for RREF(D).  The echelon's panels can stop at a row echelon form U
// (rows r x nN by pivot column, leading 1, zero below every pivot: GBLA_ECHELON_REF, which on a
// staircase D_new touches only the rows leading inside each panel's window) and the reduced
// form is then one triangular solve:
//   RREF = U_sq^-1 U,  U_sq = U[:, pc] (unit upper triangular):  RREF[:, pc] = I and
//   X = RREF[:, q] solves U_sq X = U[:, q] for the non-pivot columns q.
// Column q only involves the r_q = #{pc < q} pivot rows above it (U[i][q] = 0 for pc[i] > q),
// so the solve costs sum_q r_q (r_q - 1) / 2 modMACs, against the sum over pivot columns c of
// #{rows above} x #{all columns right of c} that a Gauss-Jordan back elimination spends
// (which also keeps the future pivot columns of earlier rows up to date).
// The solve is the K5' sweep itself: transposed and with both pivot orders reversed
// (a' = r - 1 - i), X^T U_sq^T = U[:, q]^T becomes x'_q A' = c'_q with
//   A'[a'][b'] = U[r-1-b'][pc[r-1-a']]  (upper unitriangular, dense: every band tile I <= J),
//   c'_q[a']   = U[r-1-a'][q],  lead of target q = r - r_q (targets: q descending),
// and the sweep writes x'_q[a'] straight into R[r-1-a'][q] (R = U in place: every target column
// is read into its C tiles before its batch is swept, the band tiles read pivot columns only).
namespace {

// A' band tiles, row-major A layout (element (a', b') at toff(a' % 128, b' % 128)) for k_diag_inv /
// k_ahat; pivots r .. NB*128-1 are identity (padding)
__global__ void k_bs_band(int64_t r, const uint64_t *__restrict__ tl, const uint64_t *__restrict__ offA,
                          const uint16_t *__restrict__ U, int64_t ldU, const uint32_t *__restrict__ pc,
                          uint8_t *__restrict__ tilesA)
{
    const uint64_t code = tl[blockIdx.x];
    const uint32_t I = (uint32_t)(code >> 32), J = (uint32_t)code;
    uint8_t *tile = tilesA + (offA[I] + (uint64_t)(J - I)) * TB;
    for (int it = threadIdx.x; it < 128 * 8; it += blockDim.x) {
        const uint32_t k = it & 127, c16 = (uint32_t)(it >> 7) * 16;
        const int64_t a = (int64_t)I * 128 + k;
        const uint32_t col = a < r ? pc[r - 1 - a] : 0;
        uint8_t lo[16], hi[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int64_t b = (int64_t)J * 128 + c16 + j;
            uint16_t x = 0;
            if (a < r && b < r) {
                if (a <= b) x = U[(size_t)(r - 1 - b) * ldU + col];
            } else if (a == b) {
                x = 1;
            }
            lo[j] = (uint8_t)(x & 0xff);
            hi[j] = (uint8_t)(x >> 8);
        }
        const uint32_t o = tc::toff(k, c16);
        *reinterpret_cast<uint4 *>(tile + o) = *reinterpret_cast<const uint4 *>(lo);
        *reinterpret_cast<uint4 *>(tile + PB + o) = *reinterpret_cast<const uint4 *>(hi);
    }
}

// isp[c] = 1 for pivot columns (isp has nN + 1 entries, zeroed)
__global__ void k_bs_mark(int64_t r, const uint32_t *__restrict__ pc, uint32_t *__restrict__ isp)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < r) isp[pc[k]] = 1;
}

// targets t = non-pivot columns in ascending order: q[t], lead r - #{pc < q[t]}; slot s holds target
// nq - 1 - s (leads ascending)
__global__ void k_bs_targets(int64_t nN, int64_t r, const uint32_t *__restrict__ isp,
                             const uint32_t *__restrict__ pscan, uint32_t *__restrict__ q,
                             uint32_t *__restrict__ tlead, uint32_t *__restrict__ order)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nq = nN - r;
    if (c < nN && !isp[c]) {
        const int64_t t = c - pscan[c];
        q[t] = (uint32_t)c;
        tlead[t] = (uint32_t)(r - pscan[c]);
        order[nq - 1 - t] = (uint32_t)t;
    }
}

// C tiles of the local target tiles [i0, i0 + gridDim.y): tile T, block J >= the tile's first block
__global__ void k_bs_cfill(int64_t nq, int64_t r, int64_t NB, int64_t i0, const uint32_t *__restrict__ order,
                           const uint32_t *__restrict__ tlead, const uint32_t *__restrict__ q,
                           const uint16_t *__restrict__ U, int64_t ldU, uint8_t *__restrict__ Xt)
{
    const int64_t J = blockIdx.x, li = blockIdx.y, T = i0 + li;
    const int64_t s0 = T * 128;
    if (s0 >= nq) return;
    const uint32_t l0 = tlead[order[s0]];
    if (l0 >= (uint64_t)r || J < (int64_t)(l0 / 128)) return;
    uint8_t *tile = Xt + ((size_t)li * NB + J) * TB;
    for (int it = threadIdx.x; it < 128 * 8; it += blockDim.x) {
        const uint32_t row = it & 127, c16 = (uint32_t)(it >> 7) * 16;
        const int64_t s = s0 + row;
        const bool live = s < nq;
        const uint32_t col = live ? q[order[s]] : 0;
        uint8_t lo[16], hi[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int64_t a = J * 128 + c16 + j;
            const uint16_t x = (live && a < r) ? U[(size_t)(r - 1 - a) * ldU + col] : 0;
            lo[j] = (uint8_t)(x & 0xff);
            hi[j] = (uint8_t)(x >> 8);
        }
        const uint32_t o = tc::toff(row, c16);
        *reinterpret_cast<uint4 *>(tile + o) = *reinterpret_cast<const uint4 *>(lo);
        *reinterpret_cast<uint4 *>(tile + PB + o) = *reinterpret_cast<const uint4 *>(hi);
    }
}

// RREF[i][pc[k]] = 0 for k > i (row i's entries at later pivot columns); the diagonal is 1 already
__global__ void k_bs_pivcols(int64_t r, const uint32_t *__restrict__ pc, uint16_t *__restrict__ R, int64_t ldR)
{
    const int64_t i = blockIdx.x;
    uint16_t *row = R + (size_t)i * ldR;
    for (int64_t k = i + 1 + threadIdx.x; k < r; k += blockDim.x) row[pc[k]] = 0;
}

}  // namespace

// R (rank rows, h->R / h->pivcol) from a row echelon form to the fully reduced one, in place.
gbla_status bsub_rref(gbla_mat h)
{
    cudaStream_t st = h->stream;
    const int64_t r = h->rank, nN = h->nN, ldR = h->ldR;
    if (r <= 1) return GBLA_OK;                      // nothing above any pivot
    const int64_t nq = nN - r;
    uint16_t *R = h->R;
    const uint32_t *pc = h->pivcol;
    kt_mark(h, KT_BSUB);
    if (nq > 0) {
        // targets
        uint32_t *isp, *pscan, *q, *tlead, *order;
        GBLA_TRY(dalloc_t(h, nN + 1, &isp));
        GBLA_TRY(dalloc_t(h, nN + 1, &pscan));
        GBLA_TRY(dalloc_t(h, nq, &q));
        GBLA_TRY(dalloc_t(h, nq, &tlead));
        GBLA_TRY(dalloc_t(h, nq, &order));
        GBLA_CUDA_TRY(cudaMemsetAsync(isp, 0, (nN + 1) * 4, st));
        k_bs_mark<<<grid_for(r, 256), 256, 0, st>>>(r, pc, isp);
        {
            size_t tb = 0;
            GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, isp, pscan, (int)(nN + 1), st));
            void *t;
            GBLA_TRY(dalloc(h, tb + 16, &t));
            GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t, tb, isp, pscan, (int)(nN + 1), st));
        }
        k_bs_targets<<<grid_for(nN, 256), 256, 0, st>>>(nN, r, isp, pscan, q, tlead, order);
        note_launch(2);
        GBLA_CUDA_TRY(cudaGetLastError());
        // algorithmic work: sum over targets of r_q (r_q - 1) / 2
        {
            std::vector<uint32_t> hl(nq);
            GBLA_CUDA_TRY(cudaMemcpyAsync(hl.data(), tlead, nq * 4, cudaMemcpyDeviceToHost, st));
            GBLA_CUDA_TRY(cudaStreamSynchronize(st));
            uint64_t w = 0;
            for (int64_t t = 0; t < nq; t++) {
                const uint64_t rq = (uint64_t)(r - hl[t]);
                w += rq * (rq ? rq - 1 : 0) / 2;
            }
            h->kwork[KT_BSUB] = w;
        }
        // A' band: every tile I <= J of the NB x NB block triangle
        BandTiles bt;
        bt.NB = (r + 127) / 128;
        const int64_t NB = bt.NB;
        std::vector<uint64_t> offA(NB), tl;
        std::vector<uint32_t> amax(NB, (uint32_t)(NB - 1)), jptr(NB + 1), jidx;
        uint64_t nA = 0;
        for (int64_t I = 0; I < NB; I++) { offA[I] = nA; nA += (uint64_t)(NB - I); }
        for (int64_t J = 0; J < NB; J++) {
            jptr[J] = (uint32_t)jidx.size();
            for (int64_t I = 0; I < J; I++) jidx.push_back((uint32_t)I);
        }
        jptr[NB] = (uint32_t)jidx.size();
        for (int64_t I = 0; I < NB; I++)
            for (int64_t J = I; J < NB; J++) tl.push_back(((uint64_t)I << 32) | (uint64_t)J);
        uint64_t *dtl;
        GBLA_TRY(dalloc_t(h, tl.size(), &dtl));
        GBLA_TRY(dalloc_t(h, NB, &bt.offA));
        GBLA_TRY(dalloc_t(h, NB, &bt.amax));
        GBLA_TRY(dalloc_t(h, NB + 1, &bt.jl_ptr));
        GBLA_TRY(dalloc_t(h, jidx.size() + 1, &bt.jl_idx));
        GBLA_TRY(dalloc_t(h, 3, &bt.ops));
        GBLA_TRY(dalloc(h, nA * TB + 16, (void **)&bt.tilesA));
        GBLA_TRY(dalloc(h, NB * TB + 16, (void **)&bt.invT));
        GBLA_CUDA_TRY(cudaMemcpyAsync(dtl, tl.data(), tl.size() * 8, cudaMemcpyHostToDevice, st));
        GBLA_CUDA_TRY(cudaMemcpyAsync(bt.offA, offA.data(), NB * 8, cudaMemcpyHostToDevice, st));
        GBLA_CUDA_TRY(cudaMemcpyAsync(bt.amax, amax.data(), NB * 4, cudaMemcpyHostToDevice, st));
        GBLA_CUDA_TRY(cudaMemcpyAsync(bt.jl_ptr, jptr.data(), (NB + 1) * 4, cudaMemcpyHostToDevice, st));
        if (!jidx.empty())
            GBLA_CUDA_TRY(cudaMemcpyAsync(bt.jl_idx, jidx.data(), jidx.size() * 4, cudaMemcpyHostToDevice, st));
        GBLA_CUDA_TRY(cudaMemsetAsync(bt.ops, 0, 24, st));
        k_bs_band<<<(unsigned)tl.size(), 256, 0, st>>>(r, dtl, bt.offA, R, ldR, pc, bt.tilesA);
        note_launch();
        {
            static unsigned long long attr = 0;   // devices done (dev_bit)
            if (!(attr & dev_bit())) {
                GBLA_CUDA_TRY(cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, DIAG_SMEM));
                GBLA_CUDA_TRY(cudaFuncSetAttribute(k_ahat, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TB));
                attr |= dev_bit();
            }
        }
        k_diag_inv<<<(unsigned)NB, 128, DIAG_SMEM, st>>>(h->F, bt.offA, bt.tilesA, bt.invT);
        note_launch();
        {
            // the off-diagonal tiles: the tail of each row block's list (diagonal tiles first)
            std::vector<uint64_t> off;
            for (int64_t I = 0; I < NB; I++)
                for (int64_t J = I + 1; J < NB; J++) off.push_back(((uint64_t)I << 32) | (uint64_t)J);
            if (!off.empty()) {
                uint64_t *doff;
                GBLA_TRY(dalloc_t(h, off.size(), &doff));
                GBLA_CUDA_TRY(cudaMemcpyAsync(doff, off.data(), off.size() * 8, cudaMemcpyHostToDevice, st));
                const int64_t nt = (int64_t)off.size();
                const int64_t grid = nt < 2 * (int64_t)h->ctx->sm_count ? nt : 2 * (int64_t)h->ctx->sm_count;
                k_ahat<<<(unsigned)grid, 128, 2 * TB, st>>>(h->F, NB, bt.offA, bt.amax, doff, nt, bt.tilesA, bt.invT);
                note_launch();
            }
        }
        GBLA_CUDA_TRY(cudaGetLastError());
        // target tiles in batches of X tiles
        const int64_t ntiles = (nq + 127) / 128;
        const int64_t per_tile = NB * (int64_t)TB;
        int64_t per = ntiles;
        {
            const char *e = getenv("GBLA_XT_BATCH");
            if (e && atoll(e) > 0) per = atoll(e);
            else if (ntiles * per_tile > ((int64_t)8 << 30)) {
                size_t fr = 0, tot = 0;
                if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) cudaGetLastError();
                if (h->ctx->memq) fr = h->ctx->memq(h->ctx->memq_user);
                const int64_t budget = (int64_t)fr - ((int64_t)4 << 30);
                per = budget > per_tile ? budget / per_tile : 1;
            }
            if (per > ntiles) per = ntiles;
            if (per > 65535) per = 65535;
            if (per < 1) per = 1;
        }
        GBLA_TRY(dalloc(h, (size_t)per * per_tile + 16, (void **)&bt.Xt));
        SweepSrc src;
        src.bt = &bt; src.mN = nq; src.npiv = r; src.order = order; src.tlead = tlead;
        src.Rout = R; src.ldR = ldR; src.rrev = r; src.rcol = q; src.kt = -1;   // timed as a whole
        src.group_env = "GBLA_BSUB_GROUP";
        for (int64_t i0 = 0; i0 < ntiles; i0 += per) {
            const int64_t i1 = i0 + per < ntiles ? i0 + per : ntiles;
            k_bs_cfill<<<dim3((unsigned)NB, (unsigned)(i1 - i0)), 256, 0, st>>>(nq, r, NB, i0, order, tlead, q, R, ldR,
                                                                              bt.Xt);
            note_launch();
            GBLA_CUDA_TRY(cudaGetLastError());
            GBLA_TRY(sweep_run(h, src, 0, 1, i0, i1));
        }
        GBLA_TRY(sweep_dev_err(st, "gbla_echelon_D (back substitution)"));
        unsigned long long o3[3];
        GBLA_CUDA_TRY(cudaMemcpyAsync(o3, bt.ops, 24, cudaMemcpyDeviceToHost, st));
        GBLA_CUDA_TRY(cudaStreamSynchronize(st));
        h->kexec[KT_BSUB] = o3[2] * EXEC_PER_PAIR;
        dfree(h, bt.Xt);
        dfree(h, bt.tilesA);
        dfree(h, bt.invT);
        bt.Xt = bt.tilesA = bt.invT = nullptr;
    }
    k_bs_pivcols<<<(unsigned)r, 256, 0, st>>>(r, pc, R, ldR);
    note_launch();
    kt_mark(h, KT_BSUB);
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}
