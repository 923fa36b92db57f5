// sparse_int.cu -- the sparse triangular phase on the integer pipe.
//
// K5/K6 k_reduce_targets: Alg 2 "Reduction of C and D" with the
//   multiline AXPY of Alg 1: a CTA owns one target row at a time
//   (persistent grid, targets handed out longest-first), keeps its dense
//   accumulator (u64, delayed reduction) and walks the pivot PAIRS (2k, 2k+1)
//   in ascending order.  For a pair the two scalars are
//       l1 = acc[2k],  l2 = acc[2k+1] - l1 * A[2k][2k+1]      (reading R10)
//   and one pass over the pair's union support applies both rows:
//       acc[c] += (p - l1) * v1 + (p - l2) * v2               (reading R8)
//   which is the 2x1 case of Alg 1 (two reductions per load).  The lambdas
//   are captured before the pass (reading R9), and the pass skips the pair's
//   own diagonal-block columns so the scalars of the next pair are the only
//   cross-thread dependency (one __syncthreads per pair).
//   MODE_FUSED  applies A and B parts and writes D_new = D - C A^-1 B;
//   MODE_CPRIME applies the A part only and writes C' = C A^-1;
//   MODE_FROMX  reads the lambdas from C' and applies the B part only:
//               D <- D - C' B (4-step variant).
// K8 k_trsm_cols: Step 2, B' = A^-1 B by back substitution, one
//   thread per column of B ("one only reads A and writes to B"; columns of B
//   are independent).
// K7 k_update_from_bp: Step 3, D <- D - C B'.
#include <cstring>

#include "internal.cuh"

namespace {

enum { MODE_FUSED = 0, MODE_CPRIME = 1, MODE_FROMX = 2 };

template <int MODE>
__global__ void __launch_bounds__(256) k_reduce_targets(
    int64_t mN, int64_t n, int64_t npiv, int64_t npairs, Field F, const uint32_t *__restrict__ order,
    const uint32_t *__restrict__ tlead, const uint64_t *__restrict__ cd_ptr, const uint32_t *__restrict__ cd_col,
    const uint16_t *__restrict__ cd_val, const uint64_t *__restrict__ ml_ptr, const uint32_t *__restrict__ ml_col,
    const uint32_t *__restrict__ ml_val, const uint32_t *__restrict__ ml_np, const uint32_t *__restrict__ ml_skip,
    const uint16_t *__restrict__ ml_a01, const uint32_t *__restrict__ ab_w, const uint32_t *__restrict__ ab_np,
    uint64_t *__restrict__ scratch, uint16_t *__restrict__ D, int64_t ldD, uint16_t *__restrict__ X, int64_t ldX,
    uint64_t *__restrict__ opcount, unsigned int *__restrict__ next, const uint64_t *__restrict__ mr_ptr,
    const uint64_t *__restrict__ mr_skip, const uint64_t *__restrict__ mr_np, const uint32_t *__restrict__ mr_col,
    const uint32_t *__restrict__ mr_len, const uint32_t *__restrict__ mr_rel)
{
    uint64_t *acc = scratch + (size_t)blockIdx.x * n;
    __shared__ uint32_t s_t;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int64_t nN = n - npiv;
    for (;;) {
        if (tid == 0) s_t = atomicAdd(next, 1u);
        __syncthreads();
        const uint32_t ti = s_t;
        __syncthreads();
        if (ti >= mN) break;
        const uint32_t t = order[ti];
        const uint32_t l = tlead[t];
        const int64_t k0 = (int64_t)(l < npiv ? l : npiv) / 2;   // first pair touching the lead
        const int64_t z0 = MODE == MODE_FROMX ? npiv : 2 * k0;
        for (int64_t c = z0 + tid; c < n; c += nth) acc[c] = 0;
        __syncthreads();
        if (MODE == MODE_FROMX) {
            for (int64_t c = tid; c < nN; c += nth) acc[npiv + c] = D[(size_t)t * ldD + c];
        } else {
            for (uint64_t q = cd_ptr[t] + tid; q < cd_ptr[t + 1]; q += nth) acc[cd_col[q]] = cd_val[q];
        }
        __syncthreads();
        uint64_t ops = 0;
        for (int64_t k = k0; k < npairs; k++) {
            const int64_t j0 = 2 * k, j1 = 2 * k + 1;
            uint32_t l1, l2 = 0;
            if (MODE == MODE_FROMX) {
                l1 = X[(size_t)t * ldX + j0];
                if (j1 < npiv) l2 = X[(size_t)t * ldX + j1];
            } else {
                l1 = fmod64(acc[j0], F);
                if (j1 < npiv) l2 = fmod64(acc[j1] + (uint64_t)fneg(l1, F) * ml_a01[k], F);
                if (MODE == MODE_CPRIME && tid == 0) {
                    X[(size_t)t * ldX + j0] = (uint16_t)l1;
                    if (j1 < npiv) X[(size_t)t * ldX + j1] = (uint16_t)l2;
                }
            }
            if ((l1 | l2) == 0) continue;   // uniform across the CTA (lightweight test)
            const uint64_t n1 = fneg(l1, F), n2 = fneg(l2, F);
            if (mr_ptr) {
                // column runs (GBLA_INT_RUNS=1; a warp per run, lanes over its consecutive columns):
                // one 12-byte descriptor per run instead of a 4-byte column id per slot.  Measured
                // slower on c1 (1523 vs 273 ms; a thread per run: 3159 ms): the accumulator lives in
                // global memory and the slot walk's 32 consecutive slots per warp access are the
                // coalesced ones; runs of ~8 columns leave most lanes idle
                uint64_t r0, r1;
                if (MODE == MODE_FUSED) { r0 = mr_skip[k]; r1 = mr_ptr[k + 1]; }
                else if (MODE == MODE_CPRIME) { r0 = mr_skip[k]; r1 = mr_np[k]; }
                else { r0 = mr_np[k]; r1 = mr_ptr[k + 1]; }
                const int warp = tid >> 5, lane = tid & 31, nw = nth >> 5;
                const uint32_t *vals = ml_val + ml_ptr[k];
                for (uint64_t r = r0 + warp; r < r1; r += nw) {
                    const uint32_t c0 = mr_col[r], len = mr_len[r];
                    const uint32_t *vr = vals + mr_rel[r];
                    uint64_t *ar = acc + c0;
                    for (uint32_t u = lane; u < len; u += 32) {
                        const uint32_t v = vr[u];
                        ar[u] += n1 * (v & 0xffffu) + n2 * (v >> 16);
                    }
                }
            } else {
                uint64_t q0, q1;
                if (MODE == MODE_FUSED) { q0 = ml_ptr[k] + ml_skip[k]; q1 = ml_ptr[k + 1]; }
                else if (MODE == MODE_CPRIME) { q0 = ml_ptr[k] + ml_skip[k]; q1 = ml_ptr[k] + ml_np[k]; }
                else { q0 = ml_ptr[k] + ml_np[k]; q1 = ml_ptr[k + 1]; }
                for (uint64_t q = q0 + tid; q < q1; q += nth) {
                    const uint32_t c = ml_col[q];
                    const uint32_t v = ml_val[q];
                    acc[c] += n1 * (v & 0xffffu) + n2 * (v >> 16);
                }
            }
            if (tid == 0) {
                if (MODE == MODE_FUSED) {
                    ops += (l1 ? ab_w[j0] - 1 : 0) + (l2 ? ab_w[j1] - 1 : 0);
                } else if (MODE == MODE_CPRIME) {
                    ops += (l1 ? ab_np[j0] - 1 : 0) + (l2 ? ab_np[j1] - 1 : 0);
                } else {
                    ops += (l1 ? ab_w[j0] - ab_np[j0] : 0) + (l2 ? ab_w[j1] - ab_np[j1] : 0);
                }
            }
            __syncthreads();
        }
        if (MODE != MODE_CPRIME)
            for (int64_t c = tid; c < nN; c += nth) D[(size_t)t * ldD + c] = (uint16_t)fmod64(acc[npiv + c], F);
        if (tid == 0) opcount[t] += ops;
        __syncthreads();
    }
}

// Step 2 (TRSM), one thread per column of B', rows bottom-up:
//   B'_i = B_i - sum_{j > i, A_ij != 0} A_ij B'_j.
// A row i is entries [ab_ptr[i], ab_ptr[i] + ab_np[i]) of the sigma-ordered
// pivot rows; its first entry is the diagonal 1.
__global__ void __launch_bounds__(128) k_trsm_cols(int64_t npiv, int64_t nN, Field F,
                                                   const uint64_t *__restrict__ ab_ptr,
                                                   const uint32_t *__restrict__ ab_col,
                                                   const uint16_t *__restrict__ ab_val,
                                                   const uint32_t *__restrict__ ab_np, uint16_t *__restrict__ Bp,
                                                   int64_t ld, uint64_t *__restrict__ ops_out)
{
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool live = c < nN;
    uint64_t ops = 0;
    for (int64_t i = npiv - 1; i >= 0; i--) {
        const uint64_t s = ab_ptr[i] + 1, e = ab_ptr[i] + ab_np[i];
        uint64_t acc = live ? Bp[(size_t)i * ld + c] : 0;
        uint64_t q = s;
        for (; q + 4 <= e; q += 4) {
            uint32_t j0 = ab_col[q], j1 = ab_col[q + 1], j2 = ab_col[q + 2], j3 = ab_col[q + 3];
            uint32_t a0 = fneg(ab_val[q], F), a1 = fneg(ab_val[q + 1], F);
            uint32_t a2 = fneg(ab_val[q + 2], F), a3 = fneg(ab_val[q + 3], F);
            if (live) {
                uint32_t b0 = Bp[(size_t)j0 * ld + c], b1 = Bp[(size_t)j1 * ld + c];
                uint32_t b2 = Bp[(size_t)j2 * ld + c], b3 = Bp[(size_t)j3 * ld + c];
                acc += (uint64_t)a0 * b0 + (uint64_t)a1 * b1 + (uint64_t)a2 * b2 + (uint64_t)a3 * b3;
            }
        }
        for (; q < e; q++) {
            uint32_t j = ab_col[q];
            if (live) acc += (uint64_t)fneg(ab_val[q], F) * Bp[(size_t)j * ld + c];
        }
        if (live) Bp[(size_t)i * ld + c] = (uint16_t)fmod64(acc, F);
        ops += e - s;
    }
    if (c == 0) *ops_out = ops;   // modMACs per column of B'
}

// Step 3 (standard order): D_t <- D_t - sum_{j in supp C_t} C_tj B'_j.
// Grid (targets, column chunks): the CTAs resident at one time work on consecutive targets and the
// SAME column chunk, so the B' rows they read (the targets' supports, a band that moves slowly from
// one target to the next) stay in L2 as a strip of 4 * blockDim.x columns.  Each thread owns 4
// columns (one 8-byte load per reducer row); the row's (column, coefficient) pairs are staged in
// shared memory 256 at a time; products are u32 x u32 + u64 (one IMAD.WIDE each).
__global__ void __launch_bounds__(256) k_update_from_bp(int64_t mN, int64_t nN, Field F,
                                                        const uint64_t *__restrict__ cd_ptr,
                                                        const uint32_t *__restrict__ cd_col,
                                                        const uint16_t *__restrict__ cd_val,
                                                        const uint32_t *__restrict__ cd_np,
                                                        const uint16_t *__restrict__ Bp, int64_t ldB,
                                                        uint16_t *__restrict__ D, int64_t ldD)
{
    __shared__ uint32_t s_col[256], s_a[256];
    const int tid = threadIdx.x;
    const int64_t c0 = ((int64_t)blockIdx.y * blockDim.x + tid) * 4;
    const bool live = c0 < nN;
    for (int64_t t = blockIdx.x; t < mN; t += gridDim.x) {
        uint64_t acc[4];
#pragma unroll
        for (int u = 0; u < 4; u++) acc[u] = (live && c0 + u < nN) ? D[(size_t)t * ldD + c0 + u] : 0;
        const uint64_t s = cd_ptr[t], e = s + cd_np[t];
        for (uint64_t q0 = s; q0 < e; q0 += 256) {
            const int cnt = (int)(e - q0 < 256 ? e - q0 : 256);
            __syncthreads();
            for (int i = tid; i < cnt; i += blockDim.x) {
                s_col[i] = cd_col[q0 + i];
                s_a[i] = fneg(cd_val[q0 + i], F);
            }
            __syncthreads();
            if (live) {
#pragma unroll 4
                for (int i = 0; i < cnt; i++) {
                    const uint32_t a = s_a[i];
                    // (ldB is a multiple of 128 and c0 of 4: 8-byte aligned, c0 + 3 < ldB)
                    const uint2 w = __ldg(reinterpret_cast<const uint2 *>(Bp + (size_t)s_col[i] * ldB + c0));
                    acc[0] += (uint64_t)a * (w.x & 0xffffu);
                    acc[1] += (uint64_t)a * (w.x >> 16);
                    acc[2] += (uint64_t)a * (w.y & 0xffffu);
                    acc[3] += (uint64_t)a * (w.y >> 16);
                }
            }
        }
        if (live) {
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (c0 + u < nN) D[(size_t)t * ldD + c0 + u] = (uint16_t)fmod64(acc[u], F);
        }
    }
}

__global__ void k_sum_u64(int64_t n, const uint64_t *__restrict__ a, unsigned long long *__restrict__ out)
{
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += a[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

template <int MODE>
gbla_status launch_targets(gbla_mat h)
{
    cudaStream_t st = h->stream;
    if (h->mN == 0) return GBLA_OK;
    GBLA_TRY(ensure_multilines(h));
    // GBLA_INT_RUNS=1: walk the column runs of the multilines instead of their column ids (slower, see
    // k_reduce_targets)
    const bool runs = getenv("GBLA_INT_RUNS") && atoi(getenv("GBLA_INT_RUNS")) == 1;
    int per_sm = 0;
    GBLA_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reduce_targets<MODE>, 256, 0));
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)h->ctx->sm_count * per_sm;
    if (grid > h->mN) grid = h->mN;
    uint64_t *scratch;
    unsigned int *next;
    GBLA_TRY(dalloc_t(h, (size_t)grid * h->n, &scratch));
    GBLA_TRY(dalloc_t(h, 1, &next));
    GBLA_CUDA_TRY(cudaMemsetAsync(next, 0, 4, st));
    k_reduce_targets<MODE><<<(unsigned)grid, 256, 0, st>>>(
        h->mN, h->n, h->npiv, h->npairs, h->F, h->order, h->tlead, h->cd_ptr, h->cd_col, h->cd_val, h->ml_ptr,
        h->ml_col, h->ml_val, h->ml_np, h->ml_skip, h->ml_a01, h->ab_w, h->ab_np, scratch, h->D, h->ldD, h->X, h->ldX,
        h->opcount, next, runs ? h->mr_ptr : nullptr, h->mr_skip, h->mr_np, h->mr_col, h->mr_len, h->mr_rel);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

gbla_status sum_opcount(gbla_mat h, uint64_t *out)
{
    unsigned long long *d;
    GBLA_TRY(dalloc_t(h, 1, &d));
    GBLA_CUDA_TRY(cudaMemsetAsync(d, 0, 8, h->stream));
    k_sum_u64<<<64, 256, 0, h->stream>>>(h->mN, h->opcount, d); note_launch();
    unsigned long long v = 0;
    GBLA_CUDA_TRY(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, h->stream));
    GBLA_CUDA_TRY(cudaStreamSynchronize(h->stream));
    *out = v;
    return GBLA_OK;
}

}  // namespace

gbla_status ensure_x(gbla_mat h)
{
    if (h->X) return GBLA_OK;
    h->ldX = (h->npiv + 127) / 128 * 128;
    if (h->ldX == 0) h->ldX = 128;
    size_t bytes = (size_t)(h->mN > 0 ? h->mN : 1) * h->ldX;
    GBLA_TRY(dalloc_t(h, bytes, &h->X));
    GBLA_CUDA_TRY(cudaMemsetAsync(h->X, 0, bytes * 2, h->stream));
    return GBLA_OK;
}

gbla_status reduce_c_int(gbla_mat h, bool fused, bool keep_x)
{
    if (fused) {
        if (keep_x) {
            // C' and D_new from one reduction: CPRIME pass, then FROMX pass.
            GBLA_TRY(ensure_x(h));
            GBLA_TRY(launch_targets<MODE_CPRIME>(h));
            GBLA_TRY(launch_targets<MODE_FROMX>(h));
        } else {
            GBLA_TRY(launch_targets<MODE_FUSED>(h));
        }
    } else {
        GBLA_TRY(ensure_x(h));
        GBLA_TRY(launch_targets<MODE_CPRIME>(h));
    }
    return sum_opcount(h, &h->sparse_ops);
}

gbla_status update_d_from_x_int(gbla_mat h)
{
    GBLA_TRY(launch_targets<MODE_FROMX>(h));
    return sum_opcount(h, &h->sparse_ops);
}

gbla_status reduce_b_int(gbla_mat h)
{
    cudaStream_t st = h->stream;
    h->ldB = (h->nN + 127) / 128 * 128;
    if (h->ldB == 0) h->ldB = 128;
    if (!h->Bp) GBLA_TRY(dalloc_t(h, (size_t)(h->npiv > 0 ? h->npiv : 1) * h->ldB, &h->Bp));
    GBLA_TRY(densify_impl(h, 'B', h->Bp, h->ldB));
    if (h->npiv == 0 || h->nN == 0) return GBLA_OK;
    uint64_t *ops;
    GBLA_TRY(dalloc_t(h, 1, &ops));
    k_trsm_cols<<<grid_for(h->nN, 128), 128, 0, st>>>(h->npiv, h->nN, h->F, h->ab_ptr, h->ab_col, h->ab_val,
                                                       h->ab_np, h->Bp, h->ldB, ops); note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    uint64_t v = 0;
    GBLA_CUDA_TRY(cudaMemcpyAsync(&v, ops, 8, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    h->sparse_ops += v * (uint64_t)h->nN;
    return GBLA_OK;
}

static gbla_status update_d_from_bp_rows(gbla_mat h)
{
    cudaStream_t st = h->stream;
    if (h->mN == 0 || h->nN == 0) return GBLA_OK;
    // threads per CTA = a quarter of the B' strip width in columns: 128 while the whole strip
    // (npiv rows x 1 KB) stays well inside the 126 MB L2, else 64 (c2: 1,355 -> 1,225 ms; c1/c3 the
    // same either way).  GBLA_UBP_THREADS = 64, 128 or 256 forces one.
    int nth = (size_t)h->npiv * 1024 <= ((size_t)96 << 20) ? 128 : 64;
    if (const char *e = getenv("GBLA_UBP_THREADS")) { const int v = atoi(e); if (v == 64 || v == 128 || v == 256) nth = v; }
    dim3 grid((unsigned)(h->mN < (1 << 30) ? h->mN : (1 << 30)), grid_for((h->nN + 3) / 4, nth));
    k_update_from_bp<<<grid, nth, 0, st>>>(h->mN, h->nN, h->F, h->cd_ptr, h->cd_col, h->cd_val, h->cd_np, h->Bp,
                                            h->ldB, h->D, h->ldD); note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    return GBLA_OK;
}

namespace {

// sum of a u32 array into one u64 (nnz(C) = sum of the rows' pivot-column entry counts)
__global__ void k_sum_u32(int64_t n, const uint32_t *__restrict__ a, unsigned long long *__restrict__ out)
{
    unsigned long long s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) s += a[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

}  // namespace

// Step 3 of the standard order: D -= C B'.  C is sparse, B' dense.  Two engines:
// the sparse rows of C on the INT pipe (k_update_from_bp, nnz(C) nN modMACs), or C densified and one
// K11 product on the tensor cores (mN npiv nN dense modMACs).  Measured rates on c1/c2/c3: ~5 T
// modMAC/s (INT pipe, 2/3 of its measured peak) against 150-190 T dense modMAC/s (K11 flush), so K11
// wins from a C density of ~1/34; the rule is nnz(C) >= mN npiv / 32 (c3 5.3 % -> K11; c1 2.2 % and
// c2 1.1 % -> INT).  GBLA_UPDATE_BP=int|tc forces one.
gbla_status update_d_from_bp_int(gbla_mat h)
{
    cudaStream_t st = h->stream;
    if (h->mN == 0 || h->nN == 0 || h->npiv == 0) return GBLA_OK;
    const char *e = getenv("GBLA_UPDATE_BP");
    bool dense;
    if (e && !strcmp(e, "int")) dense = false;
    else if (e && !strcmp(e, "tc")) dense = true;
    else {
        unsigned long long *d = nullptr, nnzC = 0;
        GBLA_TRY(dalloc_t(h, 1, &d));
        GBLA_CUDA_TRY(cudaMemsetAsync(d, 0, 8, st));
        k_sum_u32<<<128, 256, 0, st>>>(h->mN, h->cd_np, d); note_launch();
        GBLA_CUDA_TRY(cudaMemcpyAsync(&nnzC, d, 8, cudaMemcpyDeviceToHost, st));
        GBLA_CUDA_TRY(cudaStreamSynchronize(st));
        dfree(h, d);
        dense = (double)nnzC * 32.0 >= (double)h->mN * (double)h->npiv;
    }
    if (!dense) return update_d_from_bp_rows(h);
    uint16_t *Cd = nullptr;
    const int64_t lda = (h->npiv + 7) / 8 * 8;
    GBLA_TRY(dalloc_t(h, (size_t)h->mN * lda, &Cd));
    gbla_status s = densify_impl(h, 'C', Cd, lda);
    if (s == GBLA_OK) s = modgemm_sub_chunked(h->ctx, st, h->F, h->mN, h->nN, h->npiv, Cd, lda, h->Bp, h->ldB, h->D, h->ldD);
    if (cudaStreamSynchronize(st) != cudaSuccess && s == GBLA_OK) {
        set_error("gbla_update_D: %s", cudaGetErrorString(cudaGetLastError()));
        s = GBLA_E_CUDA;
    }
    dfree(h, Cd);
    return s;
}
