// comm.hpp -- NCCL entry points resolved at run time (dlopen), so libdogip.so
// has no link-time NCCL dependency and reuses the copy torch already loaded.
// Used for the slab interface exchange (ncclSend/ncclRecv to the z-1 / z+1
// neighbours, one grouped call per apply) and the CG scalar all-reduces.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace dogip {

struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return; }
#define DOGIP_SYM(field, name)                                           \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));   \
    if (!api.field) { api.err = std::string("missing NCCL symbol ") + name; return; }
        DOGIP_SYM(GetUniqueId, "ncclGetUniqueId")
        DOGIP_SYM(CommInitRank, "ncclCommInitRank")
        DOGIP_SYM(CommDestroy, "ncclCommDestroy")
        DOGIP_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
        DOGIP_SYM(Send, "ncclSend")
        DOGIP_SYM(Recv, "ncclRecv")
        DOGIP_SYM(GroupStart, "ncclGroupStart")
        DOGIP_SYM(GroupEnd, "ncclGroupEnd")
        DOGIP_SYM(AllReduce, "ncclAllReduce")
        DOGIP_SYM(GetErrorString, "ncclGetErrorString")
#undef DOGIP_SYM
        api.ok = true;
    });
    return api;
}

}  // namespace dogip
