// NCCL entry points resolved at run time (comm.cpp).
#pragma once

#include <cstring>

#include <nccl.h>

namespace h2b {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*get_error_string)(ncclResult_t) = nullptr;
};

// null when libnccl.so.2 cannot be opened
const NcclApi* nccl_api();
int nccl_fail(const NcclApi* api, int res, const char* what);

}  // namespace h2b
