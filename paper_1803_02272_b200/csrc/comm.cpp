#include "comm.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include <string>

#include "host_core.hpp"

namespace dsb {

Comm& Comm::get() {
    static Comm* c = new Comm();
    return *c;
}

void Comm::load() {
    if (lib_) return;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
        lib_ = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (lib_) break;
    }
    if (!lib_) throw Error(errc::internal, std::string("cannot load NCCL: ") + dlerror());
    auto sym = [&](const char* s) {
        void* p = dlsym(lib_, s);
        if (!p) throw Error(errc::internal, std::string("NCCL symbol missing: ") + s);
        return p;
    };
    getUniqueId_ = reinterpret_cast<decltype(getUniqueId_)>(sym("ncclGetUniqueId"));
    commInitRank_ = reinterpret_cast<decltype(commInitRank_)>(sym("ncclCommInitRank"));
    commDestroy_ = reinterpret_cast<decltype(commDestroy_)>(sym("ncclCommDestroy"));
    allReduce_ = reinterpret_cast<decltype(allReduce_)>(sym("ncclAllReduce"));
    broadcast_ = reinterpret_cast<decltype(broadcast_)>(sym("ncclBroadcast"));
    send_ = reinterpret_cast<decltype(send_)>(sym("ncclSend"));
    recv_ = reinterpret_cast<decltype(recv_)>(sym("ncclRecv"));
    groupStart_ = reinterpret_cast<decltype(groupStart_)>(sym("ncclGroupStart"));
    groupEnd_ = reinterpret_cast<decltype(groupEnd_)>(sym("ncclGroupEnd"));
    errorString_ = reinterpret_cast<decltype(errorString_)>(sym("ncclGetErrorString"));
}

void Comm::check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(errc::internal, std::string("NCCL error in ") + what + ": " +
                                        (errorString_ ? errorString_(r) : "?"));
}

void Comm::unique_id(void* out128) {
    load();
    ncclUniqueId id;
    check(getUniqueId_(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
}

void Comm::init(int world, int rank, const void* id128, cudaStream_t) {
    load();
    if (world < 1 || rank < 0 || rank >= world)
        throw Error(errc::invalid_argument, "bad world/rank");
    destroy();
    ncclUniqueId id;
    std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
    check(commInitRank_(&comm_, world, id, rank), "ncclCommInitRank");
    world_ = world;
    rank_ = rank;
}

void Comm::destroy() {
    if (comm_ && commDestroy_) commDestroy_(comm_);
    comm_ = nullptr;
    world_ = 1;
    rank_ = 0;
}

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t st) {
    if (!comm_) return;
    check(allReduce_(buf, buf, count, ncclFloat64, ncclSum, comm_, st), "ncclAllReduce");
}

void Comm::allreduce_max(double* buf, size_t count, cudaStream_t st) {
    if (!comm_) return;
    check(allReduce_(buf, buf, count, ncclFloat64, ncclMax, comm_, st), "ncclAllReduce");
}

void Comm::allreduce_sum_u64(unsigned long long* buf, size_t count, cudaStream_t st) {
    if (!comm_) return;
    check(allReduce_(buf, buf, count, ncclUint64, ncclSum, comm_, st), "ncclAllReduce");
}

void Comm::allgatherv(double* buf, const size_t* counts, const size_t* displs, cudaStream_t st) {
    if (!comm_ || world_ == 1) return;
    check(groupStart_(), "ncclGroupStart");
    for (int r = 0; r < world_; ++r)
        if (counts[r])
            check(broadcast_(buf + displs[r], buf + displs[r], counts[r], ncclFloat64, r, comm_, st),
                  "ncclBroadcast");
    check(groupEnd_(), "ncclGroupEnd");
}

void Comm::sendrecv(const double* sbuf, size_t count_send, int peer_send, double* rbuf,
                    size_t count_recv, int peer_recv, cudaStream_t st) {
    if (!comm_) return;
    check(groupStart_(), "ncclGroupStart");
    if (count_send) check(send_(sbuf, count_send, ncclFloat64, peer_send, comm_, st), "ncclSend");
    if (count_recv) check(recv_(rbuf, count_recv, ncclFloat64, peer_recv, comm_, st), "ncclRecv");
    check(groupEnd_(), "ncclGroupEnd");
}

void shard_rows(size_t n, int world, int rank, size_t& begin, size_t& end) {
    const size_t nb = (n + kRowPad - 1) / kRowPad;
    const size_t b0 = nb * static_cast<size_t>(rank) / static_cast<size_t>(world);
    const size_t b1 = nb * static_cast<size_t>(rank + 1) / static_cast<size_t>(world);
    begin = std::min(n, b0 * kRowPad);
    end = std::min(n, b1 * kRowPad);
}

}  // namespace dsb
