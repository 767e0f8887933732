// nccl_api.h -- NCCL entry points resolved at run time (internal).
//
// The library does not link NCCL: the sharded entry binds to whichever
// libnccl.so.2 the process already has (torch's bundled copy in a PyTorch
// process, the caller's in a C++ program) and dlopen()s it otherwise.  Only the
// handful of NCCL 2.x calls the sharded ID needs are declared here, with the
// ABI types of nccl.h (ncclUniqueId is 128 bytes; ncclFloat64 = 8).
#pragma once

#include <cstddef>
#include <string>

#include <cuda_runtime.h>

namespace idk {

typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
    char internal[128];
};
typedef int ncclResult_t;  // ncclSuccess = 0, ncclInProgress = 7
constexpr int kNcclUint8 = 1;
constexpr int kNcclInt32 = 2;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclMin = 3;

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    int (*GetVersion)(int*) = nullptr;
};

// nullptr (and *err set) when no libnccl.so.2 can be found or a symbol is missing.
const NcclApi* nccl_api(std::string* err);

}  // namespace idk
