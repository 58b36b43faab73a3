// Data-parallel plumbing of the training step: images shard across GPUs
// (one process per GPU), and the step's one exchange is the sum of the fp32 gradient arena
// over ranks -- ncclAllReduce over NVLink / NVSwitch on the model's stream (capturable, so it
// sits inside the step's CUDA graph between the backward and AdamW).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", reusing the copy torch already loaded when
// there is one): the library has no link-time NCCL dependency and single-GPU use never touches
// it.  Only the handful of entry points below are resolved.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace affmae_b200 {
namespace {

// nccl.h types, declared locally (ABI-stable since NCCL 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
constexpr int kNcclFloat32 = 7;  // ncclFloat32
constexpr int kNcclSum = 0;      // ncclSum

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        n.h = h;
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    });
    return n;
}

int nccl_fail(ncclResult_t r, const char* what) {
    const char* s = nccl().error_string ? nccl().error_string(r) : "?";
    return fail(AFFMAE_ECUDA, std::string(what) + ": " + s);
}

int require() {
    Nccl& n = nccl();
    if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.all_reduce || !n.comm_destroy)
        return fail(AFFMAE_EUNSUPPORTED, "NCCL (libnccl.so.2) not available");
    return AFFMAE_OK;
}

}  // namespace

int nccl_unique_id(uint8_t* out128) {
    if (!out128) return fail(AFFMAE_ECONFIG, "nccl_unique_id: null pointer");
    if (int rc = require()) return rc;
    ncclUniqueId id;
    if (ncclResult_t r = nccl().get_unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
    return AFFMAE_OK;
}

int nccl_comm_init(const uint8_t* id128, int nranks, int rank, void** comm) {
    if (!id128 || !comm) return fail(AFFMAE_ECONFIG, "nccl_comm_init: null pointer");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(AFFMAE_ECONFIG, "nccl_comm_init: bad rank");
    if (int rc = require()) return rc;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    if (ncclResult_t r = nccl().comm_init_rank(&c, nranks, id, rank)) return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return AFFMAE_OK;
}

int nccl_allreduce_sum_f32(void* comm, float* buf, int64_t n, cudaStream_t st) {
    if (int rc = require()) return rc;
    if (ncclResult_t r = nccl().all_reduce(buf, buf, size_t(n), kNcclFloat32, kNcclSum,
                                           static_cast<ncclComm_t>(comm), st))
        return nccl_fail(r, "ncclAllReduce");
    return AFFMAE_OK;
}

void nccl_comm_destroy(void* comm) {
    if (comm && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

}  // namespace affmae_b200
