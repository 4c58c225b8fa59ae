// comm.cu -- the one collective of the multi-GPU step (BASELINE config 4): an NCCL all-gather of the
// packed preconditioned gradients over NVLink/NVSwitch, behind the C-ABI.
//
// libnccl is resolved at run time (dlopen "libnccl.so.2", reusing an already-loaded copy -- e.g. the one torch.
// distributed brought in -- before loading the system one), so the library loads and runs its single-GPU paths on
// hosts without NCCL; NCCL failures surface as RKFAC_NCCL_ERROR.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "comm.cuh"
#include "engine.cuh"

namespace rkfac_b200 {

namespace {

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        r.all_gather = reinterpret_cast<decltype(r.all_gather)>(dlsym(h, "ncclAllGather"));
        r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
        return r;
    }();
    RKFAC_REQUIRE(n.get_unique_id && n.comm_init_rank && n.all_gather && n.comm_destroy, RKFAC_NCCL_ERROR,
                  "libnccl.so.2 not found (NCCL is needed for the multi-GPU all-gather)");
    return n;
}

void check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const char* s = nccl().error_string ? nccl().error_string(r) : "";
    throw Error(RKFAC_NCCL_ERROR, std::string(what) + ": " + s);
}

}  // namespace

size_t nccl_unique_id_bytes() { return sizeof(ncclUniqueId); }

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

void* nccl_comm_init(const void* id_bytes, int nranks, int rank) {
    RKFAC_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, RKFAC_INVALID_ARGUMENT, "bad NCCL rank / size");
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    ncclComm_t c = nullptr;
    check(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
    return c;
}

void nccl_comm_destroy(void* comm) {
    if (comm) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

void nccl_allgather(void* comm, const float* send, float* recv, long long count, cudaStream_t s) {
    RKFAC_REQUIRE(comm, RKFAC_INVALID_ARGUMENT, "no NCCL communicator attached to the context");
    check(nccl().all_gather(send, recv, (size_t)count, ncclFloat32, static_cast<ncclComm_t>(comm), s),
          "ncclAllGather");
}

}  // namespace rkfac_b200
