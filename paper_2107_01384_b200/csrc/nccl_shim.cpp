// NCCL for the sharded compress, loaded at run time: the
// process's libnccl.so.2 (the one torch already mapped, else the system one)
// is opened once and the few entry points used here are resolved from it, so
// the library neither pins an NCCL version nor conflicts with torch's copy.
#include "nccl_shim.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

namespace tcb {

namespace {

struct Nccl {
    using GetUniqueId = ncclResult_t (*)(ncclUniqueId*);
    using CommInitRank = ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int);
    using CommDestroy = ncclResult_t (*)(ncclComm_t);
    using AllReduce = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                       cudaStream_t);
    using AllGather = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    using ErrorString = const char* (*)(ncclResult_t);
    GetUniqueId get_unique_id = nullptr;
    CommInitRank comm_init_rank = nullptr;
    CommDestroy comm_destroy = nullptr;
    AllReduce all_reduce = nullptr;
    AllGather all_gather = nullptr;
    ErrorString error_string = nullptr;
    std::string err;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl o;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            o.err = std::string("nccl: cannot load libnccl.so.2: ") + (e ? e : "?");
            return o;
        }
        o.get_unique_id = reinterpret_cast<Nccl::GetUniqueId>(dlsym(h, "ncclGetUniqueId"));
        o.comm_init_rank = reinterpret_cast<Nccl::CommInitRank>(dlsym(h, "ncclCommInitRank"));
        o.comm_destroy = reinterpret_cast<Nccl::CommDestroy>(dlsym(h, "ncclCommDestroy"));
        o.all_reduce = reinterpret_cast<Nccl::AllReduce>(dlsym(h, "ncclAllReduce"));
        o.all_gather = reinterpret_cast<Nccl::AllGather>(dlsym(h, "ncclAllGather"));
        o.error_string = reinterpret_cast<Nccl::ErrorString>(dlsym(h, "ncclGetErrorString"));
        if (!o.get_unique_id || !o.comm_init_rank || !o.comm_destroy || !o.all_reduce || !o.all_gather)
            o.err = "nccl: libnccl.so.2 lacks an entry point";
        return o;
    }();
    return n;
}

void check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const Nccl& n = nccl();
    throw Error(std::string("nccl: ") + what + " failed: " + (n.error_string ? n.error_string(r) : "?"));
}

const Nccl& need() {
    const Nccl& n = nccl();
    if (!n.err.empty()) throw Error(n.err);
    return n;
}

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    check(need().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
}

void* nccl_comm_init(const unsigned char id[128], int world, int rank) {
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    ncclComm_t c = nullptr;
    check(need().comm_init_rank(&c, world, u, rank), "ncclCommInitRank");
    return c;
}

void nccl_comm_destroy(void* comm) {
    if (comm) need().comm_destroy(static_cast<ncclComm_t>(comm));
}

void nccl_allreduce_sum_f64(double* buf, u64 count, void* comm, cudaStream_t s) {
    check(need().all_reduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s),
          "ncclAllReduce");
}

void nccl_allgather_f64(const double* send, double* recv, u64 count_per_rank, void* comm, cudaStream_t s) {
    check(need().all_gather(send, recv, count_per_rank, ncclFloat64, static_cast<ncclComm_t>(comm), s),
          "ncclAllGather");
}

}  // namespace tcb
