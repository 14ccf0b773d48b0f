// Minimal dlopen binding of NCCL (libnccl.so.2): the process may already have
// torch's bundled NCCL loaded, in which case dlopen returns that instance.
// Types and enums come from the system nccl.h (2.27); only stable core API
// entry points are used.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace qtb {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static NcclApi& get() {
        static NcclApi api;
        static bool tried = false;
        if (!tried) {
            tried = true;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
            if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (h) {
#define QTB_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
                QTB_NCCL_SYM(GetUniqueId);
                QTB_NCCL_SYM(CommInitRank);
                QTB_NCCL_SYM(CommDestroy);
                QTB_NCCL_SYM(AllGather);
                QTB_NCCL_SYM(AllReduce);
                QTB_NCCL_SYM(ReduceScatter);
                QTB_NCCL_SYM(Send);
                QTB_NCCL_SYM(Recv);
                QTB_NCCL_SYM(GroupStart);
                QTB_NCCL_SYM(GroupEnd);
                QTB_NCCL_SYM(GetErrorString);
#undef QTB_NCCL_SYM
                api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.AllReduce && api.Send &&
                         api.Recv && api.GroupStart && api.GroupEnd;
            }
        }
        return api;
    }
};

}  // namespace qtb
