// nccl_dyn.cu -- NCCL for the partitioned phase engine, bound at run time.
//
// libplv does not link NCCL: the first multi-GPU call dlopen()s the
// libnccl.so.2 already mapped into the process (torch's), else the system
// one.  Single-GPU use never touches NCCL.  The communicator is created from
// a unique id the caller distributes (rank 0 -> all, over torch.distributed),
// one rank per process / GPU.
#include "nccl_dyn.cuh"
#include <dlfcn.h>
#include <mutex>

namespace plv {

namespace {
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_api;
std::once_flag g_once;

void load() {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
        g_api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
        if (g_api.h) break;
    }
    for (const char *nm : names) {
        if (g_api.h) break;
        g_api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!g_api.h) return;
#define PLV_SYM(f, s) *(void **)(&g_api.f) = dlsym(g_api.h, s)
    PLV_SYM(getUniqueId, "ncclGetUniqueId");
    PLV_SYM(commInitRank, "ncclCommInitRank");
    PLV_SYM(commDestroy, "ncclCommDestroy");
    PLV_SYM(broadcast, "ncclBroadcast");
    PLV_SYM(allReduce, "ncclAllReduce");
    PLV_SYM(allGather, "ncclAllGather");
    PLV_SYM(groupStart, "ncclGroupStart");
    PLV_SYM(groupEnd, "ncclGroupEnd");
    PLV_SYM(getErrorString, "ncclGetErrorString");
#undef PLV_SYM
}

const NcclApi &api() {
    std::call_once(g_once, load);
    if (!g_api.h || !g_api.getUniqueId || !g_api.commInitRank || !g_api.broadcast ||
        !g_api.groupStart || !g_api.groupEnd)
        PLV_FAIL(PLV_ECUDA, "NCCL (libnccl.so.2) is not available to libplv");
    return g_api;
}

void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) {
        const char *msg = g_api.getErrorString ? g_api.getErrorString(r) : "?";
        PLV_FAIL(PLV_ECUDA, "%s: NCCL error %d (%s)", what, (int)r, msg);
    }
}
}  // namespace

void nccl_group_start() { nccl_check(api().groupStart(), "ncclGroupStart"); }
void nccl_group_end() { nccl_check(api().groupEnd(), "ncclGroupEnd"); }

void nccl_bcast_inplace(void *buf, size_t count, ncclDataType_t type, int root, void *comm,
                        cudaStream_t s) {
    nccl_check(api().broadcast(buf, buf, count, type, root, (ncclComm_t)comm, s), "ncclBroadcast");
}

void nccl_allgather_inplace(void *buf, size_t bytes_per_rank, int rank, void *comm,
                            cudaStream_t s) {
    const NcclApi &a = api();
    if (!a.allGather) PLV_FAIL(PLV_ECUDA, "ncclAllGather is not available");
    nccl_check(a.allGather((const char *)buf + (size_t)rank * bytes_per_rank, buf, bytes_per_rank,
                           ncclUint8, (ncclComm_t)comm, s),
               "ncclAllGather");
}

}  // namespace plv

extern "C" int plv_nccl_unique_id(uint8_t *id_h) {
    PLV_ENTRY
    ncclUniqueId id;
    plv::nccl_check(plv::api().getUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == PLV_NCCL_ID_BYTES, "ncclUniqueId size");
    memcpy(id_h, &id, sizeof(id));
    PLV_EXIT
}

extern "C" int plv_nccl_comm_init(int64_t rank, int64_t world, const uint8_t *id_h,
                                  void **comm_h) {
    PLV_ENTRY
    if (world < 1 || rank < 0 || rank >= world) PLV_FAIL(PLV_EINVAL, "bad rank/world");
    ncclUniqueId id;
    memcpy(&id, id_h, sizeof(id));
    ncclComm_t c = nullptr;
    plv::nccl_check(plv::api().commInitRank(&c, (int)world, id, (int)rank), "ncclCommInitRank");
    *comm_h = (void *)c;
    PLV_EXIT
}

extern "C" int plv_nccl_comm_destroy(void *comm) {
    PLV_ENTRY
    if (comm) plv::nccl_check(plv::api().commDestroy((ncclComm_t)comm), "ncclCommDestroy");
    PLV_EXIT
}
