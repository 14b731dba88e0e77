// nccl_shim.h -- NCCL entry points resolved at run time (dlopen "libnccl.so.2").
//
// The library must load on a CPU-only box (tests check its exports) and inside a
// process where PyTorch already loaded its own libnccl.so.2; RTLD_NOLOAD reuses that
// copy, otherwise the system library is opened.  Only the x-slab multi-GPU path calls it.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace cg {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
};

inline const NcclApi &nccl_real() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.send = (decltype(a.send))dlsym(h, "ncclSend");
        a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
        a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
        a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.send && a.recv && a.allReduce && a.groupStart &&
               a.groupEnd;
        return a;
    }();
    return api;
}

// The active table: the real libnccl, or a test transport installed with nccl_set_active()
// (nccl_loopback.h via cg_nccl_loopback).
inline const NcclApi *&nccl_active() {
    static const NcclApi *p = nullptr;
    return p;
}
inline const NcclApi &nccl() {
    const NcclApi *p = nccl_active();
    return p ? *p : nccl_real();
}

}  // namespace cg
