// dist.cu -- multi-GPU plumbing of libgbla over NCCL (NVLink 5 / NVSwitch).
//
// The NCCL communicator is built inside the library from a 128-byte
// ncclUniqueId that the caller distributes (the Python binding uses
// torch.distributed for that), so the C ABI carries no torch or NCCL types.
#include <nccl.h>

#include "internal.cuh"

#define GBLA_NCCL_TRY(expr)                                                                \
    do {                                                                                   \
        ncclResult_t r_ = (expr);                                                          \
        if (r_ != ncclSuccess) {                                                           \
            set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(r_)); \
            return GBLA_E_NCCL;                                                            \
        }                                                                                  \
    } while (0)

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
    if (world == 1) return GBLA_OK;
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
