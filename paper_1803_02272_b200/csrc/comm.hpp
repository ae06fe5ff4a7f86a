// Multi-GPU plumbing: one process per GPU. Two transports behind one
// interface:
//   * NCCL over NVLink / NVSwitch (the product transport), loaded with dlopen
//     at communicator creation (no link-time dependency; the process's
//     already-loaded libnccl.so.2 — e.g. torch's — is reused);
//   * a host-staged TCP transport (DSB_COMM_TRANSPORT=host when the id is
//     created): every collective synchronizes the stream, copies the device
//     buffer to the host, exchanges it through rank 0 over loopback sockets
//     and copies the result back. It exists so that several ranks can run
//     the real sharded code on ONE GPU in tests (no kernel ever waits on
//     another process — the ranks meet only in blocking host calls); it is
//     not a compute path.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace dsb {

class Comm {
public:
    enum class Mode { none, nccl, host };
    static Comm& get();
    bool active() const { return mode_ != Mode::none; }
    Mode mode() const { return mode_; }
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
    // in place: rank r contributes buf[r * count, (r + 1) * count) (ncclAllGather)
    void allgather(double* buf, size_t count, cudaStream_t st);
    // rank r contributes counts[r] elements at displs[r] of buf (in place)
    void allgatherv(double* buf, const size_t* counts, const size_t* displs, cudaStream_t st);
    // pairwise exchange: send `count_send` to peer_send, receive `count_recv` from peer_recv
    void sendrecv(const double* sbuf, size_t count_send, int peer_send, double* rbuf,
                  size_t count_recv, int peer_recv, cudaStream_t st);

private:
    Comm() = default;
    void load();
    void check(ncclResult_t r, const char* what);
    Mode mode_ = Mode::none;
    int world_ = 1, rank_ = 0;

    // ---- NCCL ----
    void* lib_ = nullptr;
    ncclComm_t comm_ = nullptr;
    ncclResult_t (*getUniqueId_)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank_)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy_)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce_)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather_)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*broadcast_)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*send_)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                          cudaStream_t) = nullptr;
    ncclResult_t (*recv_)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart_)() = nullptr;
    ncclResult_t (*groupEnd_)() = nullptr;
    const char* (*errorString_)(ncclResult_t) = nullptr;

    // ---- host-staged transport (star through rank 0) ----
    int listen_fd_ = -1;       // rank 0, between unique_id and init
    std::vector<int> peers_;   // rank 0: socket of rank r (r >= 1); others: [0] = rank 0
    std::vector<unsigned char> stage_;
    void host_send(int fd, const void* p, size_t bytes);
    void host_recv(int fd, void* p, size_t bytes);
    // D2H of `bytes` at dev into stage_ (after a stream sync)
    unsigned char* host_stage_in(const void* dev, size_t bytes, cudaStream_t st);
    template <typename T, typename Op>
    void host_allreduce(T* buf, size_t count, cudaStream_t st, Op op);
};

// Row shard of rank `rank` among `world`: 256-row blocks in equal runs of
// B = ceil(blocks / world) (the last rank takes the remainder, possibly
// none), so every shard boundary is a panel-block boundary and the panel
// all-gather moves one equal-size chunk per rank (ncclAllGather).
void shard_rows(size_t n, int world, int rank, size_t& begin, size_t& end);
// rows of one rank's panel chunk (B blocks of 256) and the padded panel
// height world * chunk
size_t shard_chunk_rows(size_t n, int world);

}  // namespace dsb
