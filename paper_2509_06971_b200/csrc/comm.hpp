// comm.hpp -- halo exchange and reductions for the slab decomposition.
//
// A rank owns node planes [kb, ke) of the outermost axis and stores one ghost plane
// on each interior face; planes are contiguous in HBM, so a halo is one
// px*ny-double block per component.  Two transports share the same schedule:
//   * NCCL (one process per GPU): send/recv to the +-1 ranks inside one group,
//     all-reduce for the scalars.  libnccl is dlopen'ed (the process may already
//     hold torch's copy; reusing it avoids two NCCLs in one address space).
//   * local group (one process driving several contexts, e.g. several GPUs or one
//     GPU in tests): each context pulls its ghost planes from its neighbours'
//     owned planes with stream-ordered peer copies.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>

namespace petto_b200 {

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    bool load(std::string& err) {
        if (handle) return true;
        // PETTO_NCCL_LIB names another libnccl-compatible library (the tests' in-process
        // multi-rank emulator); otherwise prefer an NCCL already mapped into the process
        // (torch's), then the loader path
        if (const char* lib = std::getenv("PETTO_NCCL_LIB")) handle = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
        if (!handle) handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!handle) handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!handle) handle = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!handle) {
            err = "libnccl.so.2 not found";
            return false;
        }
        auto sym = [&](const char* n) { return dlsym(handle, n); };
        GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
        CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
        CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
        Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
        Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
        AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
        Broadcast = reinterpret_cast<decltype(Broadcast)>(sym("ncclBroadcast"));
        GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
        GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
        GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
        if (!GetUniqueId || !CommInitRank || !Send || !Recv || !AllReduce || !Broadcast || !GroupStart || !GroupEnd) {
            err = "libnccl.so.2 lacks the point-to-point / collective API";
            return false;
        }
        return true;
    }
};

inline NcclApi& nccl() {
    static NcclApi api;
    return api;
}

}  // namespace petto_b200
