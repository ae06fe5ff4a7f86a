// Multi-GPU plumbing: one process per GPU, NCCL over NVLink / NVSwitch,
// loaded with dlopen at communicator creation (no link-time dependency; the
// process's already-loaded libnccl.so.2 — e.g. torch's — is reused).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>

namespace dsb {

class Comm {
public:
    static Comm& get();
    bool active() const { return comm_ != nullptr; }
    int world() const { return world_; }
    int rank() const { return rank_; }

    void unique_id(void* out128);
    void init(int world, int rank, const void* id128, cudaStream_t st);
    void destroy();

    // collectives on the library stream (double elements)
    void allreduce_sum(double* buf, size_t count, cudaStream_t st);
    void allreduce_max(double* buf, size_t count, cudaStream_t st);
    // sum of unsigned 64-bit integers (wraps mod 2^64)
    void allreduce_sum_u64(unsigned long long* buf, size_t count, cudaStream_t st);
    // rank r contributes counts[r] elements at displs[r] of buf (in place)
    void allgatherv(double* buf, const size_t* counts, const size_t* displs, cudaStream_t st);
    // pairwise exchange: send `count_send` to peer_send, receive `count_recv` from peer_recv
    void sendrecv(const double* sbuf, size_t count_send, int peer_send, double* rbuf,
                  size_t count_recv, int peer_recv, cudaStream_t st);

private:
    Comm() = default;
    void load();
    void check(ncclResult_t r, const char* what);
    void* lib_ = nullptr;
    ncclComm_t comm_ = nullptr;
    int world_ = 1, rank_ = 0;
    // dlsym'd entry points
    ncclResult_t (*getUniqueId_)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank_)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy_)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce_)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*broadcast_)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*send_)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                          cudaStream_t) = nullptr;
    ncclResult_t (*recv_)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart_)() = nullptr;
    ncclResult_t (*groupEnd_)() = nullptr;
    const char* (*errorString_)(ncclResult_t) = nullptr;
};

// Row shard of rank `rank` among `world`: the reference's chunk formula
// (ref src/parallel.hpp:33-34) applied to 256-row blocks, so every shard
// boundary is a panel-block boundary: rows [256 nb r / W, 256 nb (r+1) / W).
void shard_rows(size_t n, int world, int rank, size_t& begin, size_t& end);

}  // namespace dsb
