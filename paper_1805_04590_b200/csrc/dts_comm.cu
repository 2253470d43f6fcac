// dts_comm.cu -- the row-band exchange transport (multi-GPU section of DESIGN.md).
//
// The only collective of the path is an all-gather of the per-rank band tuples of a
// column pass (5 floats per column for a 1-channel target).  Two transports:
//  - NCCL (one process per GPU, NVLink/NVSwitch): ncclAllGather on the launch stream.
//    NCCL is resolved at run time with dlopen (torch's bundled libnccl.so.2 is usually
//    already loaded in the process), so the library has no link-time NCCL dependency.
//  - loopback: N ranks as N host threads of one process on one GPU (tests): the ranks
//    rendezvous on a host barrier and copy each other's device buffers.  Kernels never
//    wait on one another; only the host threads do.
#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dts_comm.h"

namespace dts {

namespace {

struct NcclApi {
    bool ok = false;
    std::string err;
    int (*getUniqueId)(void*) = nullptr;
    int (*commInitRank)(void**, int, NcclUniqueId, int) = nullptr;
    int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    const char* (*getErrorString)(int) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already loaded (torch)?
        if (!h) {
            const char* p = std::getenv("DTS_NCCL_LIB");
            if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = "libnccl.so.2 not found (set DTS_NCCL_LIB)";
            return;
        }
        api.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclGetUniqueId"));
        api.commInitRank = reinterpret_cast<int (*)(void**, int, NcclUniqueId, int)>(dlsym(h, "ncclCommInitRank"));
        api.allGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
            dlsym(h, "ncclAllGather"));
        api.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(h, "ncclCommDestroy"));
        api.getErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy;
        if (!api.ok) api.err = "libnccl.so.2 lacks the expected symbols";
    });
    return api;
}

constexpr int kNcclFloat32 = 7;  // ncclDataType_t ncclFloat32 (stable across NCCL 2.x)

}  // namespace

struct LoopGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    unsigned long long gen = 0;
    std::vector<const float*> send;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long my = gen;
        if (++count == n) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != my; });
        }
    }
};

bool nccl_unique_id(void* id128, std::string* err) {
    NcclApi& a = nccl();
    if (!a.ok) {
        *err = a.err;
        return false;
    }
    int r = a.getUniqueId(id128);
    if (r != 0) {
        *err = a.getErrorString ? a.getErrorString(r) : "ncclGetUniqueId failed";
        return false;
    }
    return true;
}

Comm* comm_nccl(const void* id128, int rank, int nranks, std::string* err) {
    NcclApi& a = nccl();
    if (!a.ok) {
        *err = a.err;
        return nullptr;
    }
    NcclUniqueId id;
    std::memcpy(id.internal, id128, sizeof(id.internal));
    void* c = nullptr;
    int r = a.commInitRank(&c, nranks, id, rank);
    if (r != 0) {
        *err = a.getErrorString ? a.getErrorString(r) : "ncclCommInitRank failed";
        return nullptr;
    }
    Comm* cm = new Comm();
    cm->kind = Comm::NCCL;
    cm->rank = rank;
    cm->nranks = nranks;
    cm->nccl = c;
    return cm;
}

std::vector<Comm*> comm_loopback(int nranks) {
    auto g = std::make_shared<LoopGroup>();
    g->n = nranks;
    g->send.assign(nranks, nullptr);
    std::vector<Comm*> out;
    for (int r = 0; r < nranks; ++r) {
        Comm* cm = new Comm();
        cm->kind = Comm::LOOPBACK;
        cm->rank = r;
        cm->nranks = nranks;
        cm->group = g;
        out.push_back(cm);
    }
    return out;
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->kind == Comm::NCCL && c->nccl && nccl().ok) nccl().commDestroy(c->nccl);
    delete c;
}

// recv[q * count + i] = send_q[i] for every rank q (rank order), on `s`
bool comm_allgather(Comm* c, const float* send, float* recv, size_t count, cudaStream_t s, std::string* err) {
    if (c->kind == Comm::NCCL) {
        int r = nccl().allGather(send, recv, count, kNcclFloat32, c->nccl, s);
        if (r != 0) {
            *err = nccl().getErrorString ? nccl().getErrorString(r) : "ncclAllGather failed";
            return false;
        }
        return true;
    }
    LoopGroup& g = *c->group;
    cudaError_t e = cudaStreamSynchronize(s);  // our send buffer is complete
    if (e != cudaSuccess) {
        *err = cudaGetErrorString(e);
        return false;
    }
    g.send[c->rank] = send;
    g.barrier();
    for (int q = 0; q < g.n && e == cudaSuccess; ++q)
        e = cudaMemcpyAsync(recv + (size_t)q * count, g.send[q], count * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    g.barrier();  // nobody overwrites a send buffer before every rank has copied it
    if (e != cudaSuccess) {
        *err = cudaGetErrorString(e);
        return false;
    }
    return true;
}

}  // namespace dts
