// comm.cu -- the one collective of the path: the
// row-sharded trace(A*B) of config 5b ends with a sum all-reduce of one
// float64 over NCCL (NVLink / NVSwitch).  The library talks to NCCL itself,
// so the product path never routes its data through torch.distributed; the
// host layer only has to move the 128-byte unique id from rank 0 to the
// other ranks (any rendezvous will do: torch.distributed's object
// broadcast, a file, MPI).
//
// NCCL is resolved at run time (dlopen), preferring the copy already loaded
// in the process (torch ships one): two NCCL builds in one process would
// not share state.  Semantics of the reduced value: the sum of the ranks'
// trace_of_product partials, lazymat/kernels.py:157-164 per shard.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace lm {
namespace {

struct NcclApi {
    void *handle = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commInitAll)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*getVersion)(int *) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
};

std::mutex g_mu;
NcclApi g_api;

int load_api(const char *path) {
    std::lock_guard<std::mutex> lock(g_mu);
    if (g_api.handle) return 0;
    void *h = nullptr;
    if (path && path[0]) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        set_error("NCCL not found (%s)", dlerror());
        return -1;
    }
    NcclApi a;
    a.handle = h;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(h, "ncclCommInitAll"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.getVersion = reinterpret_cast<decltype(a.getVersion)>(dlsym(h, "ncclGetVersion"));
    a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.getUniqueId || !a.commInitRank || !a.commInitAll || !a.allReduce || !a.commDestroy || !a.getVersion) {
        set_error("NCCL library lacks an expected symbol");
        return -1;
    }
    g_api = a;
    return 0;
}

#define LM_NCCL(call)                                                                                           \
    do {                                                                                                        \
        ncclResult_t _r = (call);                                                                               \
        if (_r != ncclSuccess) {                                                                                \
            ::lm::set_error("%s: NCCL error %d (%s)", #call, (int)_r,                                           \
                            g_api.getErrorString ? g_api.getErrorString(_r) : "");                              \
            return -3;                                                                                          \
        }                                                                                                       \
    } while (0)

}  // namespace
}  // namespace lm

using namespace lm;

extern "C" {

int lm_nccl_load(const char *path, int *version_out) {
    clear_error();
    if (int rc = load_api(path)) return rc;
    if (version_out) LM_NCCL(g_api.getVersion(version_out));
    return 0;
}

int lm_nccl_unique_id(uint8_t *id_out) {
    clear_error();
    LM_REQUIRE(id_out != nullptr, "nccl_unique_id: null output");
    if (int rc = load_api(nullptr)) return rc;
    ncclUniqueId id;
    LM_NCCL(g_api.getUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == LM_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return 0;
}

int lm_nccl_init_rank(int nranks, int rank, const uint8_t *id, void **comm_out) {
    clear_error();
    LM_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "nccl_init_rank: rank %d of %d", rank, nranks);
    LM_REQUIRE(id != nullptr && comm_out != nullptr, "nccl_init_rank: null argument");
    if (int rc = load_api(nullptr)) return rc;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    LM_NCCL(g_api.commInitRank(&c, nranks, uid, rank));  // on the calling thread's current device
    *comm_out = c;
    return 0;
}

int lm_nccl_init_all(int ndev, const int *devs, void **comms_out) {
    clear_error();
    LM_REQUIRE(ndev >= 1 && comms_out != nullptr, "nccl_init_all: bad arguments");
    if (int rc = load_api(nullptr)) return rc;
    LM_NCCL(g_api.commInitAll(reinterpret_cast<ncclComm_t *>(comms_out), ndev, devs));
    return 0;
}

int lm_allreduce_sum(void *comm, int dtype, void *d_buf, int64_t count, void *stream) {
    clear_error();
    LM_REQUIRE(comm != nullptr, "allreduce_sum: null communicator");
    LM_REQUIRE(dtype == LM_F64 || dtype == LM_F32, "allreduce_sum: bad dtype");
    LM_REQUIRE(count >= 0, "allreduce_sum: negative count");
    if (count == 0) return 0;
    if (int rc = load_api(nullptr)) return rc;
    LM_NCCL(g_api.allReduce(d_buf, d_buf, (size_t)count, dtype == LM_F64 ? ncclFloat64 : ncclFloat32, ncclSum,
                            static_cast<ncclComm_t>(comm), as_stream(stream)));
    return 0;
}

int lm_allreduce_sum_f64(void *comm, double *d_val, void *stream) {
    return lm_allreduce_sum(comm, LM_F64, d_val, 1, stream);
}

int lm_nccl_destroy(void *comm) {
    clear_error();
    if (!comm) return 0;
    if (int rc = load_api(nullptr)) return rc;
    LM_NCCL(g_api.commDestroy(static_cast<ncclComm_t>(comm)));
    return 0;
}

}  // extern "C"
