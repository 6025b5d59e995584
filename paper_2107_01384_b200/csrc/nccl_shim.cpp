// NCCL for the sharded compress, loaded at run time: the
// process's libnccl.so.2 (the one torch already mapped, else the system one)
// is opened once and the few entry points used here are resolved from it, so
// the library neither pins an NCCL version nor conflicts with torch's copy.
#include "nccl_shim.hpp"
#include "pipeline.hpp"

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

void nccl_allgather_bytes(const void* send, void* recv, u64 bytes_per_rank, void* comm, cudaStream_t s) {
    check(need().all_gather(send, recv, bytes_per_rank, ncclUint8, static_cast<ncclComm_t>(comm), s),
          "ncclAllGather");
}

// ---------------------------------------------------------------- ShardComm
void ShardComm::allreduce_sum_f64(double* d, u64 n, cudaStream_t s) const {
    if (!host) {
        nccl_allreduce_sum_f64(d, n, comm, s);
        return;
    }
    std::vector<double> h(n);
    d2h(h.data(), d, n * sizeof(double), s);
    stream_sync(s);
    if (host->allreduce_sum_f64(host->ctx, h.data(), n) != 0) throw Error("sharded compress: host all-reduce failed");
    TCB_CUDA(cudaMemcpyAsync(d, h.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    stream_sync(s);
}

void ShardComm::allgather(const void* dsend, void* drecv, u64 bytes, cudaStream_t s) const {
    if (!host) {
        nccl_allgather_bytes(dsend, drecv, bytes, comm, s);
        return;
    }
    std::vector<u8> hs(bytes), hr(bytes * static_cast<u64>(world));
    if (bytes) d2h(hs.data(), dsend, bytes, s);
    stream_sync(s);
    if (host->allgather(host->ctx, hs.data(), hr.data(), bytes) != 0)
        throw Error("sharded compress: host all-gather failed");
    if (!hr.empty()) TCB_CUDA(cudaMemcpyAsync(drecv, hr.data(), hr.size(), cudaMemcpyHostToDevice, s));
    stream_sync(s);
}

std::vector<std::vector<u8>> ShardComm::allgather_blobs(const std::vector<u8>& mine, cudaStream_t s) const {
    // sizes first, then every blob padded to the largest
    std::vector<std::vector<u8>> out(world);
    if (world == 1) {
        out[0] = mine;
        return out;
    }
    DevBuf<u64> ds(1, s), dsa(world, s);
    const u64 sz = mine.size();
    ds.upload(&sz, 1);
    allgather(ds.p, dsa.p, sizeof(u64), s);
    const auto sizes = dsa.to_host();
    u64 mx = 0;
    for (u64 v : sizes) mx = std::max(mx, v);
    if (mx == 0) return out;
    DevBuf<u8> send(mx, s), recv(mx * world, s);
    if (sz) send.upload(mine.data(), sz);
    allgather(send.p, recv.p, mx, s);
    std::vector<u8> all(mx * world);
    recv.download(all.data(), all.size());
    stream_sync(s);
    for (int r = 0; r < world; ++r) out[r].assign(all.begin() + r * mx, all.begin() + r * mx + sizes[r]);
    return out;
}

}  // namespace tcb
