// NCCL for row-sharded plans (one plan per device plus a
// communicator; the x all-gather of every sharded matvec runs inside
// h2b_matvec_sharded).  NCCL is opened at first use (dlopen libnccl.so.2 --
// the copy PyTorch already loaded when there is one), so libh2b.so has no
// link-time NCCL dependency and single-GPU users never touch it.

#include <dlfcn.h>

#include <mutex>

#include <cuda_runtime.h>
#include <nccl.h>

#include "h2b_internal.h"
#include "nccl_api.h"

#define H2B_CUDA_TRY(expr)                                                                          \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return h2b::fail(H2B_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
    } while (0)

namespace h2b {

namespace {
NcclApi g_api;
bool g_tried = false;
std::mutex g_mu;
}  // namespace

const NcclApi* nccl_api() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_tried) {
        g_tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            g_api.get_unique_id = reinterpret_cast<decltype(g_api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
            g_api.comm_init_rank = reinterpret_cast<decltype(g_api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
            g_api.comm_destroy = reinterpret_cast<decltype(g_api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
            g_api.all_gather = reinterpret_cast<decltype(g_api.all_gather)>(dlsym(h, "ncclAllGather"));
            g_api.get_error_string =
                reinterpret_cast<decltype(g_api.get_error_string)>(dlsym(h, "ncclGetErrorString"));
            g_api.ok = g_api.get_unique_id && g_api.comm_init_rank && g_api.comm_destroy && g_api.all_gather &&
                       g_api.get_error_string;
        }
    }
    return g_api.ok ? &g_api : nullptr;
}

int nccl_fail(const NcclApi* api, int res, const char* what) {
    return fail(H2B_ERR_CUDA, std::string(what) + ": " + api->get_error_string(static_cast<ncclResult_t>(res)));
}

}  // namespace h2b

using namespace h2b;

extern "C" int h2b_comm_unique_id(void* h_id) {
    if (!h_id) return fail(H2B_ERR_INVALID, "h2b_comm_unique_id: null pointer");
    const NcclApi* api = nccl_api();
    if (!api) return fail(H2B_ERR_INVALID, "h2b_comm_unique_id: libnccl.so.2 not found");
    ncclUniqueId id;
    const ncclResult_t r = api->get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == H2B_COMM_ID_BYTES, "unique id size");
    std::memcpy(h_id, &id, sizeof(id));
    return ok();
}

extern "C" int h2b_comm_init(void** comm, int nranks, const void* h_id, int rank, int device) {
    if (!comm || !h_id || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(H2B_ERR_INVALID, "h2b_comm_init: bad argument");
    const NcclApi* api = nccl_api();
    if (!api) return fail(H2B_ERR_INVALID, "h2b_comm_init: libnccl.so.2 not found");
    H2B_CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, h_id, sizeof(id));
    ncclComm_t c = nullptr;
    const ncclResult_t r = api->comm_init_rank(&c, nranks, id, rank);
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommInitRank");
    *comm = c;
    return ok();
}

extern "C" int h2b_comm_destroy(void* comm) {
    if (!comm) return ok();
    const NcclApi* api = nccl_api();
    if (!api) return fail(H2B_ERR_INVALID, "h2b_comm_destroy: libnccl.so.2 not found");
    const ncclResult_t r = api->comm_destroy(static_cast<ncclComm_t>(comm));
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommDestroy");
    return ok();
}
