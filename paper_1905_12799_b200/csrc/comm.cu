// comm.cu — native NCCL communicator for the sharded paths.
//
// The two exchanges north_star names run on the engine stream with no host round trip:
//   * k-means partial sums / counts (sampler.py:94-115 per Lloyd iteration): kt_lloyd_run
//     enqueues pass -> ncclAllReduce(int64) -> apply, several passes per host check;
//   * the PPO gradient all-reduce (agent.py:245-257 per epoch) and the round's reward /
//     advantage statistics: kt_comm_all_reduce_f64 has the kt_collective callback signature,
//     so kt_search_round_ex calls NCCL directly (no Python in the loop).
// NCCL is loaded with dlopen("libnccl.so.2") on first use — in a torch process that is the
// library torch.distributed already loaded — so the engine library itself has no link-time
// NCCL dependency.  The unique id travels between ranks over the caller's process group.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace kt {
namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.error_string;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(KT_ERR_INTERNAL, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace
}  // namespace kt

struct kt_comm {
    ncclComm_t comm = nullptr;
    kt_engine* engine = nullptr;
    int rank = 0, world = 1;
};

namespace kt {
// all-reduce SUM in place on the communicator's engine stream (used by kt_lloyd_run)
void comm_all_reduce_i64(kt_comm* c, int64_t* buf, int64_t count) {
    nccl_check(nccl().all_reduce(buf, buf, size_t(count), ncclInt64, ncclSum, c->comm, c->engine->stream),
               "ncclAllReduce");
}
}  // namespace kt

extern "C" {

int kt_comm_unique_id(uint8_t* id_out) {
    KT_API_BEGIN
    using namespace kt;
    if (!nccl().ok) fail(KT_ERR_UNSUPPORTED, nccl().why);
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    KT_API_END
}

int kt_comm_create(kt_engine* e, const uint8_t* id, int rank, int world, kt_comm** out) {
    KT_API_BEGIN
    using namespace kt;
    if (!nccl().ok) fail(KT_ERR_UNSUPPORTED, nccl().why);
    if (world < 1 || rank < 0 || rank >= world) fail(KT_ERR_VALUE, "bad rank / world size");
    KT_CUDA(cudaSetDevice(e->device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    auto* c = new kt_comm;
    c->engine = e;
    c->rank = rank;
    c->world = world;
    const ncclResult_t r = nccl().comm_init_rank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        nccl_check(r, "ncclCommInitRank");
    }
    *out = c;
    KT_API_END
}

int kt_comm_destroy(kt_comm* c) {
    KT_API_BEGIN
    if (c) {
        if (c->comm) kt::nccl().comm_destroy(c->comm);
        delete c;
    }
    KT_API_END
}

// kt_all_reduce_f64_fn-compatible: user = kt_comm*, buf on the communicator's engine stream
int kt_comm_all_reduce_f64(void* user, double* dev_buf, int64_t count) {
    KT_API_BEGIN
    using namespace kt;
    auto* c = static_cast<kt_comm*>(user);
    nccl_check(nccl().all_reduce(dev_buf, dev_buf, size_t(count), ncclFloat64, ncclSum, c->comm, c->engine->stream),
               "ncclAllReduce");
    KT_API_END
}

int kt_comm_all_reduce_i64(kt_comm* c, int64_t* dev_buf, int64_t count) {
    KT_API_BEGIN
    kt::comm_all_reduce_i64(c, dev_buf, count);
    KT_API_END
}

}  // extern "C"
