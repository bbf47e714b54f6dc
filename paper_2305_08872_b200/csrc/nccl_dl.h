// nccl_dl.h — the few NCCL entry points the backend uses (nccl.h surface),
// resolved at run time with dlopen so the library has no link-time NCCL
// dependency; inside a torch process this returns torch's own libnccl.so.2.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstddef>
#include <mutex>
#include <type_traits>

namespace amltk {

using ncclComm_t = struct ncclComm*;
constexpr int kNcclSuccess = 0;
constexpr int kNcclUint8 = 1;
constexpr int kNcclUniqueIdBytes = 128;
struct NcclUniqueId {
    char internal[kNcclUniqueIdBytes];
};

struct Nccl {
    int (*init_all)(ncclComm_t*, int, const int*) = nullptr;
    int (*get_unique_id)(NcclUniqueId*) = nullptr;
    int (*init_rank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
    int (*bcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*group_start)() = nullptr;
    int (*group_end)() = nullptr;
    int (*destroy)(ncclComm_t) = nullptr;
    const char* (*err)(int) = nullptr;
    bool ok = false;
};

inline const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](auto& fp, const char* name) { fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(h, name)); };
        sym(n.init_all, "ncclCommInitAll");
        sym(n.get_unique_id, "ncclGetUniqueId");
        sym(n.init_rank, "ncclCommInitRank");
        sym(n.bcast, "ncclBroadcast");
        sym(n.group_start, "ncclGroupStart");
        sym(n.group_end, "ncclGroupEnd");
        sym(n.destroy, "ncclCommDestroy");
        sym(n.err, "ncclGetErrorString");
        n.ok = n.init_all && n.get_unique_id && n.init_rank && n.bcast && n.group_start && n.group_end &&
               n.destroy;
    });
    return n;
}

inline const char* nccl_error_string(int r) { return nccl().err ? nccl().err(r) : "NCCL error"; }

}  // namespace amltk
