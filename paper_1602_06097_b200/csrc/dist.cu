// dist.cu -- multi-GPU path of libgbla over NCCL (NVLink 5 / NVSwitch).
//
// The NCCL communicator is built inside the library from a 128-byte
// ncclUniqueId that the caller distributes (the Python binding uses
// torch.distributed for that), so the C ABI carries no torch or NCCL types.
//
// gbla_reduce with a communicator of G ranks (new order):
//   C1  rank 0's CSR is broadcast to every rank (ncclBroadcast of the sizes,
//       then row_ptr / col / val); every rank splices it (deterministic, so
//       the A|B band tiles are replicated).
//   --  the target tiles (128 targets each, sorted by lead) are dealt
//       cyclically: rank g owns tiles g, g+G, ...  (the work per tile falls
//       with its lead, so cyclic dealing balances the triangular profile);
//       each rank runs the tensor-core sweep and update on its tiles only -
//       targets are independent, no communication.
//   C5  ncclAllReduce of the two modMAC counters.
//   --  D_new stays row-sharded (each rank holds the rows of its tiles); the
//       echelon is distributed (panel.cu: panels_dist): per
//       panel an all-reduce of lead counts, an all-gather of the candidates'
//       slices, the same panel factorization on every rank, an all-reduce of
//       the selected rows and a local trailing update; R is assembled by
//       broadcasts of every rank's pivot rows.
// GBLA_DIST_EMULATE=G (no communicator) runs the G shards one after the
// other on one GPU (one shared D whose rows the ranks split) and replaces the
// collectives by device copies / sums: the same partition, kernels and data
// movement, a local transport.
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include "internal.cuh"

#define GBLA_NCCL_TRY(expr)                                                                \
    do {                                                                                   \
        ncclResult_t r_ = (expr);                                                          \
        if (r_ != ncclSuccess) {                                                           \
            set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(r_)); \
            return GBLA_E_NCCL;                                                            \
        }                                                                                  \
    } while (0)

void band_release(gbla_mat h);
gbla_status tc_shard(gbla_mat h, int prank, int pworld);

// Asynchronous NCCL failures (a peer died, a network error) surface only through
// ncclCommGetAsyncError: polled at every point where the host waits for a distributed phase.
// On an error the communicator is aborted (every pending collective returns) and the call fails.
gbla_status dist_check_async(gbla_ctx ctx)
{
    if (!ctx->nccl_comm) return GBLA_OK;
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError((ncclComm_t)ctx->nccl_comm, &ar);
    if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
        set_error("NCCL asynchronous error: %s", ncclGetErrorString(r != ncclSuccess ? r : ar));
        ncclCommAbort((ncclComm_t)ctx->nccl_comm);
        ctx->nccl_comm = nullptr;
        ctx->world = 1;
        ctx->rank = 0;
        return GBLA_E_NCCL;
    }
    return GBLA_OK;
}
gbla_status tc_read_ops(gbla_mat h, unsigned long long ops[2]);
int64_t tc_ntiles(gbla_mat h);
unsigned long long *tc_ops_dev(gbla_mat h);

void dist_destroy(gbla_ctx ctx)
{
    if (ctx->nccl_comm) {
        ncclCommDestroy((ncclComm_t)ctx->nccl_comm);
        ctx->nccl_comm = nullptr;
    }
    ctx->rank = 0;
    ctx->world = 1;
}

gbla_status dist_set_comm(gbla_ctx ctx, const void *id, int rank, int world)
{
    dist_destroy(ctx);
    if (!id) return GBLA_OK;                  // detach
    // world == 1 with an id: a one-rank communicator, so the distributed code path (row-sharded
    // sparse phase, distributed echelon) and every NCCL call in it run on one GPU (tests)
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
    memcpy(&uid, id, sizeof uid);
    GBLA_CUDA_TRY(cudaSetDevice(ctx->device));
    ncclComm_t comm;
    GBLA_NCCL_TRY(ncclCommInitRank(&comm, world, uid, rank));
    ctx->nccl_comm = comm;
    ctx->rank = rank;
    ctx->world = world;
    return GBLA_OK;
}

extern "C" gbla_status gbla_nccl_get_unique_id(void *out128)
{
    if (!out128) { set_error("NULL output"); return GBLA_E_INVAL; }
    ncclUniqueId uid;
    GBLA_NCCL_TRY(ncclGetUniqueId(&uid));
    memcpy(out128, &uid, sizeof uid);
    return GBLA_OK;
}


int dist_emulated_world()
{
    const char *e = getenv("GBLA_DIST_EMULATE");
    if (!e) return 1;
    const int g = atoi(e);
    return g > 1 ? g : 1;
}

// C1: broadcast rank 0's CSR (device or host arrays) to every rank; returns a
// device CSR view valid on this rank (owned by h).
gbla_status dist_bcast_input(gbla_mat h, const gbla_csr *M, bool host_input, gbla_csr *out, gbla_status root_ok)
{
    gbla_ctx ctx = h->ctx;
    ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
    cudaStream_t st = h->stream;
    int64_t *ddims;
    GBLA_TRY(dalloc_t(h, 4, &ddims));
    // hd[3]: rank 0's validation status of M (every rank returns it)
    int64_t hd[4] = {ctx->rank == 0 ? M->m : 0, ctx->rank == 0 ? M->n : 0, ctx->rank == 0 ? M->nnz : 0,
                     ctx->rank == 0 ? (int64_t)root_ok : 0};
    GBLA_CUDA_TRY(cudaMemcpyAsync(ddims, hd, 32, cudaMemcpyHostToDevice, st));
    GBLA_NCCL_TRY(ncclBroadcast(ddims, ddims, 4, ncclInt64, 0, comm, st));
    GBLA_CUDA_TRY(cudaMemcpyAsync(hd, ddims, 32, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    GBLA_TRY(dist_check_async(ctx));
    if (hd[3] != GBLA_OK) {
        if (ctx->rank != 0) set_error("gbla_splice: rank 0 rejected the input matrix (status %lld)", (long long)hd[3]);
        return (gbla_status)hd[3];
    }
    const int64_t m = hd[0], n = hd[1], nnz = hd[2];
    uint64_t *rp;
    uint32_t *col;
    uint16_t *val;
    GBLA_TRY(dalloc_t(h, m + 1, &rp));
    GBLA_TRY(dalloc_t(h, nnz, &col));
    GBLA_TRY(dalloc_t(h, nnz, &val));
    if (ctx->rank == 0) {
        const cudaMemcpyKind k = host_input ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        GBLA_CUDA_TRY(cudaMemcpyAsync(rp, M->row_ptr, (m + 1) * 8, k, st));
        if (nnz) {
            GBLA_CUDA_TRY(cudaMemcpyAsync(col, M->col, nnz * 4, k, st));
            GBLA_CUDA_TRY(cudaMemcpyAsync(val, M->val, nnz * 2, k, st));
        }
    }
    GBLA_NCCL_TRY(ncclGroupStart());
    GBLA_NCCL_TRY(ncclBroadcast(rp, rp, m + 1, ncclUint64, 0, comm, st));
    if (nnz) {
        GBLA_NCCL_TRY(ncclBroadcast(col, col, nnz, ncclUint32, 0, comm, st));
        GBLA_NCCL_TRY(ncclBroadcast(val, val, nnz * 2, ncclUint8, 0, comm, st));
    }
    GBLA_NCCL_TRY(ncclGroupEnd());
    out->m = m; out->n = n; out->nnz = nnz;
    out->row_ptr = rp; out->col = col; out->val = val;
    return GBLA_OK;
}

// sparse phase of this rank's shard (or of every emulated shard), op-count
// all-reduce, D_new all-gather.
gbla_status dist_sparse_phase(gbla_mat h)
{
    gbla_ctx ctx = h->ctx;
    cudaStream_t st = h->stream;
    const bool real = ctx->nccl_comm != nullptr;
    const int G = real ? ctx->world : dist_emulated_world();
    const int me = real ? ctx->rank : 0;
    if (h->mN == 0 || h->npiv == 0) return GBLA_OK;   // D_new = D on every rank
    if (real) {
        GBLA_TRY(tc_shard(h, me, G));
    } else {
        for (int g = 0; g < G; g++) GBLA_TRY(tc_shard(h, g, G));
    }
    band_release(h);
    // C5: modMAC counters (each rank counted its own tiles)
    unsigned long long ops[2];
    GBLA_TRY(tc_read_ops(h, ops));            // this rank's tiles (kernel work for the roofline)
    h->kwork[KT_SWEEP] = ops[0];
    h->kwork[KT_UPDATE] = ops[1];
    if (real) {
        unsigned long long *d = tc_ops_dev(h);
        GBLA_NCCL_TRY(ncclAllReduce(d, d, 2, ncclUint64, ncclSum, (ncclComm_t)ctx->nccl_comm, st));
    }
    GBLA_TRY(tc_read_ops(h, ops));
    h->sparse_ops = ops[0] + ops[1];
    GBLA_TRY(sweep_dev_err(st, "gbla_reduce (sharded sparse phase)"));
    if (real) GBLA_TRY(dist_check_async(ctx));
    // D_new stays row-sharded: the echelon is distributed (panel.cu: panels_dist)
    return GBLA_OK;
}

// ---- replicated echelon: D_new all-gathered, then the single-GPU echelon on every rank ----------
// Echelon mode of a multi-GPU reduction (GBLA_DIST_ECHELON): "replicated" (default) gathers D_new
// so that every rank holds all of it and runs the single-GPU echelon (the K14 / super-panel /
// look-ahead routes, no per-panel collective or host synchronization; identical R on every rank
// since every step is deterministic); "panels" keeps D row-sharded and runs the distributed panel
// Gauss-Jordan (panel.cu: panels_dist; per panel an all-reduce, an all-gather and a host sync).
bool dist_echelon_replicated()
{
    const char *e = getenv("GBLA_DIST_ECHELON");
    return !(e && strcmp(e, "panels") == 0);
}

namespace {
// Dp[slot] = D[order[slot]] for the slots of this rank's target tiles (T = me + G i); block = one slot
__global__ void k_pack_own(int64_t mN, int64_t ldD, const uint16_t *__restrict__ D, const uint32_t *__restrict__ order,
                           int me, int G, uint16_t *__restrict__ Dp)
{
    const int64_t l = blockIdx.x, T = me + (int64_t)G * (l / 128), slot = T * 128 + l % 128;
    if (slot >= mN) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(D + (size_t)order[slot] * ldD);
    uint4 *dst = reinterpret_cast<uint4 *>(Dp + (size_t)slot * ldD);
    for (int64_t q = threadIdx.x; q < ldD / 8; q += blockDim.x) dst[q] = src[q];
}
// D[order[slot]] = Dp[slot] for every slot of the other ranks' tiles
__global__ void k_unpack_others(int64_t mN, int64_t ldD, const uint16_t *__restrict__ Dp,
                                const uint32_t *__restrict__ order, int me, int G, uint16_t *__restrict__ D)
{
    const int64_t slot = blockIdx.x;
    if ((slot / 128) % G == me) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(Dp + (size_t)slot * ldD);
    uint4 *dst = reinterpret_cast<uint4 *>(D + (size_t)order[slot] * ldD);
    for (int64_t q = threadIdx.x; q < ldD / 8; q += blockDim.x) dst[q] = __ldcs(src + q);
}
}  // namespace

// C7 (replicated echelon): every rank ends with all of D_new.  The target tiles (128 slots of the
// lead order each) were dealt cyclically, so round k = tiles kG .. kG+G-1 is one contiguous block
// of the slot-ordered buffer Dp in which rank g holds sub-block g: one in-place ncclAllGather per
// round (grouped), between a pack of this rank's rows into slot order and an unpack of the others'
// rows back into D's row order.  Extra memory: one D-sized buffer while the gather runs (c4:
// 45 GB; the band tiles are released by then).  If a rank cannot allocate it, every rank learns
// it (all-reduce of a flag) and D stays row-sharded (panels_dist).  Emulated ranks share one
// fully updated D: nothing to move.
gbla_status dist_gather_dnew(gbla_mat h)
{
    gbla_ctx ctx = h->ctx;
    const bool real = ctx->nccl_comm != nullptr;
    if (!real) { h->dist_rows = false; return GBLA_OK; }
    if (h->mN == 0 || h->nN == 0 || h->npiv == 0) { h->dist_rows = false; return GBLA_OK; }
    ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
    cudaStream_t st = h->stream;
    const int G = ctx->world, me = ctx->rank;
    const int64_t mN = h->mN, ldD = h->ldD;
    const int64_t ntile = (mN + 127) / 128, rounds = (ntile + G - 1) / G;
    uint16_t *Dp = nullptr;
    uint32_t *fail;
    GBLA_TRY(dalloc_t(h, 1, &fail));
    const gbla_status as = dalloc_t(h, (size_t)rounds * G * 128 * ldD, &Dp);
    const uint32_t hf = as == GBLA_OK ? 0u : 1u;
    GBLA_CUDA_TRY(cudaMemcpyAsync(fail, &hf, 4, cudaMemcpyHostToDevice, st));
    GBLA_NCCL_TRY(ncclAllReduce(fail, fail, 1, ncclUint32, ncclSum, comm, st));
    uint32_t nfail = 0;
    GBLA_CUDA_TRY(cudaMemcpyAsync(&nfail, fail, 4, cudaMemcpyDeviceToHost, st));
    GBLA_CUDA_TRY(cudaStreamSynchronize(st));
    GBLA_TRY(dist_check_async(ctx));
    dfree(h, fail);
    if (nfail) {                              // some rank is short of memory: keep D row-sharded
        if (Dp) dfree(h, Dp);
        return GBLA_OK;
    }
    const int64_t own = ((ntile - me + G - 1) / G) * 128;   // slots of this rank's tiles (padded)
    if (own > 0) k_pack_own<<<(unsigned)own, 256, 0, st>>>(mN, ldD, h->D, h->order, me, G, Dp);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    const size_t blk = (size_t)128 * ldD;    // u16 per tile
    GBLA_NCCL_TRY(ncclGroupStart());
    for (int64_t k = 0; k < rounds; k++) {
        uint16_t *round = Dp + (size_t)k * G * blk;
        GBLA_NCCL_TRY(ncclAllGather(round + (size_t)me * blk, round, blk * 2, ncclUint8, comm, st));
    }
    GBLA_NCCL_TRY(ncclGroupEnd());
    k_unpack_others<<<(unsigned)mN, 256, 0, st>>>(mN, ldD, Dp, h->order, me, G, h->D);
    note_launch();
    GBLA_CUDA_TRY(cudaGetLastError());
    dfree(h, Dp);
    GBLA_TRY(dist_check_async(ctx));
    h->dist_rows = false;
    return GBLA_OK;
}

// ---- transport of the distributed echelon (NCCL, on the handle's stream) ---------
gbla_status dist_allreduce_u32(gbla_mat h, uint32_t *buf, size_t n)
{
    GBLA_NCCL_TRY(ncclAllReduce(buf, buf, n, ncclUint32, ncclSum, (ncclComm_t)h->ctx->nccl_comm, h->stream));
    return GBLA_OK;
}
gbla_status dist_allreduce_u64(gbla_mat h, unsigned long long *buf, size_t n)
{
    GBLA_NCCL_TRY(ncclAllReduce(buf, buf, n, ncclUint64, ncclSum, (ncclComm_t)h->ctx->nccl_comm, h->stream));
    return GBLA_OK;
}
gbla_status dist_allgather(gbla_mat h, const void *send, void *recv, size_t bytes)
{
    GBLA_NCCL_TRY(ncclAllGather(send, recv, bytes, ncclUint8, (ncclComm_t)h->ctx->nccl_comm, h->stream));
    return GBLA_OK;
}
gbla_status dist_bcast(gbla_mat h, void *buf, size_t bytes, int root)
{
    GBLA_NCCL_TRY(ncclBroadcast(buf, buf, bytes, ncclUint8, root, (ncclComm_t)h->ctx->nccl_comm, h->stream));
    return GBLA_OK;
}
