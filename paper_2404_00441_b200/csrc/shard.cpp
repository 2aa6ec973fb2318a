// shard.cpp -- NCCL plumbing of candidate-position sharding.
// libnccl.so.2 is loaded on first use (dlopen), so the library itself has no
// link-time NCCL dependency: a process that already holds torch's bundled
// NCCL gets that one (same soname), a plain C++ caller gets the system one.
// Only four entry points are needed: the unique id, communicator init and
// destroy, and the per-wave all-gather of the shards' top-K records.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "internal.hpp"

namespace ccwgpu {
namespace {

// nccl.h types restated (the header is not needed to build): ncclResult_t is
// an int enum, ncclComm_t an opaque pointer, ncclUniqueId 128 bytes,
// ncclUint8 = 1 in ncclDataType_t.
using nccl_result = int;
struct nccl_id {
    char internal[128];
};
constexpr int kNcclUint8 = 1;

struct NcclApi {
    nccl_result (*get_unique_id)(nccl_id*) = nullptr;
    nccl_result (*comm_init_rank)(void** comm, int nranks, nccl_id id, int rank) = nullptr;
    nccl_result (*comm_destroy)(void* comm) = nullptr;
    nccl_result (*all_gather)(const void* send, void* recv, size_t count, int dtype, void* comm,
                              cudaStream_t st) = nullptr;
    const char* (*error_string)(nccl_result) = nullptr;
    std::string load_error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_gather)
            api.load_error = "libnccl.so.2 lacks a required symbol";
    });
    if (!api.load_error.empty()) throw Fail(CCW_ERR_CUDA, api.load_error);
    return api;
}

void check(nccl_result r, const char* what) {
    if (r != 0) {
        const NcclApi& a = nccl();
        throw Fail(CCW_ERR_CUDA, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
    }
}

}  // namespace

void nccl_unique_id(uint8_t* out128) {
    nccl_id id;
    check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, sizeof id.internal);
}

void* nccl_comm_init(int nranks, int rank, const uint8_t* id128) {
    nccl_id id;
    std::memcpy(id.internal, id128, sizeof id.internal);
    void* comm = nullptr;
    check(nccl().comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
    return comm;
}

void nccl_comm_destroy(void* comm) {
    if (comm) nccl().comm_destroy(comm);
}

void nccl_all_gather_bytes(void* comm, const void* send, void* recv, size_t bytes, cudaStream_t st) {
    check(nccl().all_gather(send, recv, bytes, kNcclUint8, comm, st), "ncclAllGather");
}

}  // namespace ccwgpu
