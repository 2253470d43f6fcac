// dts_comm.h -- row-band exchange transport (internal).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

namespace dts {

struct NcclUniqueId {
    char internal[128];
};

struct LoopGroup;

struct Comm {
    enum Kind { NCCL = 0, LOOPBACK = 1 } kind = NCCL;
    int rank = 0, nranks = 1;
    void* nccl = nullptr;               // ncclComm_t
    std::shared_ptr<LoopGroup> group;   // loopback
};

bool nccl_unique_id(void* id128, std::string* err);
Comm* comm_nccl(const void* id128, int rank, int nranks, std::string* err);
std::vector<Comm*> comm_loopback(int nranks);
void comm_destroy(Comm* c);
bool comm_allgather(Comm* c, const float* send, float* recv, size_t count, cudaStream_t s, std::string* err);

}  // namespace dts
