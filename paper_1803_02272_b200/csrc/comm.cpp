#include "comm.hpp"

#include <arpa/inet.h>
#include <dlfcn.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "host_core.hpp"

namespace dsb {

namespace {

constexpr char kHostMagic[8] = {'D', 'S', 'B', 'H', 'O', 'S', 'T', '1'};

bool host_transport_requested() {
    const char* e = std::getenv("DSB_COMM_TRANSPORT");
    return e && std::strcmp(e, "host") == 0;
}

// every host-transport message starts with this header, so ranks that call
// different collectives fail loudly instead of misreading each other's bytes
struct MsgHdr {
    uint32_t tag;
    int32_t a, b;
    uint64_t bytes;
};

enum : uint32_t { kTagReduce = 0x52454431, kTagGather = 0x47415431, kTagSendRecv = 0x53525631 };

}  // namespace

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
    allGather_ = reinterpret_cast<decltype(allGather_)>(sym("ncclAllGather"));
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
    if (host_transport_requested()) {
        // rank 0 (this process) listens on a loopback port; the id carries it
        if (listen_fd_ >= 0) close(listen_fd_);
        listen_fd_ = socket(AF_INET, SOCK_STREAM, 0);
        if (listen_fd_ < 0) throw Error(errc::internal, "host transport: socket() failed");
        sockaddr_in a{};
        a.sin_family = AF_INET;
        a.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
        a.sin_port = 0;
        socklen_t len = sizeof(a);
        if (bind(listen_fd_, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0 ||
            listen(listen_fd_, 64) != 0 ||
            getsockname(listen_fd_, reinterpret_cast<sockaddr*>(&a), &len) != 0)
            throw Error(errc::internal, "host transport: cannot listen on 127.0.0.1");
        unsigned char id[128] = {};
        std::memcpy(id, kHostMagic, 8);
        std::memcpy(id + 8, &a.sin_port, 2);
        std::memcpy(id + 12, &a.sin_addr.s_addr, 4);
        std::memcpy(out128, id, 128);
        return;
    }
    load();
    ncclUniqueId id;
    check(getUniqueId_(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
}

void Comm::init(int world, int rank, const void* id128, cudaStream_t) {
    if (world < 1 || rank < 0 || rank >= world)
        throw Error(errc::invalid_argument, "bad world/rank");
    destroy();
    const unsigned char* id = static_cast<const unsigned char*>(id128);
    if (std::memcmp(id, kHostMagic, 8) == 0) {
        uint16_t port;
        uint32_t addr;
        std::memcpy(&port, id + 8, 2);
        std::memcpy(&addr, id + 12, 4);
        peers_.assign(rank == 0 ? world : 1, -1);
        if (rank == 0) {
            if (listen_fd_ < 0)
                throw Error(errc::invalid_argument,
                            "host transport: rank 0 must be the process that created the id");
            for (int k = 1; k < world; ++k) {
                pollfd pf{listen_fd_, POLLIN, 0};
                if (poll(&pf, 1, 120000) != 1)
                    throw Error(errc::internal, "host transport: peers did not connect in 120 s");
                const int fd = accept(listen_fd_, nullptr, nullptr);
                if (fd < 0) throw Error(errc::internal, "host transport: accept failed");
                int32_t r = -1;
                host_recv(fd, &r, 4);
                if (r < 1 || r >= world || peers_[r] >= 0)
                    throw Error(errc::internal, "host transport: bad peer rank");
                peers_[r] = fd;
            }
            close(listen_fd_);
            listen_fd_ = -1;
        } else {
            sockaddr_in a{};
            a.sin_family = AF_INET;
            a.sin_port = port;
            a.sin_addr.s_addr = addr;
            int fd = -1;
            const auto t0 = std::chrono::steady_clock::now();
            for (;;) {
                fd = socket(AF_INET, SOCK_STREAM, 0);
                if (fd >= 0 && connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof(a)) == 0) break;
                if (fd >= 0) close(fd);
                if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
                    throw Error(errc::internal, "host transport: cannot reach rank 0");
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
            const int32_t r = rank;
            host_send(fd, &r, 4);
            peers_[0] = fd;
        }
        for (int fd : peers_)
            if (fd >= 0) {
                int one = 1;
                setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
                // a peer that died or never arrives ends the wait with an error
                timeval tv{600, 0};
                setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
            }
        mode_ = Mode::host;
        world_ = world;
        rank_ = rank;
        return;
    }
    load();
    ncclUniqueId nid;
    std::memcpy(nid.internal, id128, NCCL_UNIQUE_ID_BYTES);
    check(commInitRank_(&comm_, world, nid, rank), "ncclCommInitRank");
    mode_ = Mode::nccl;
    world_ = world;
    rank_ = rank;
}

void Comm::destroy() {
    if (comm_ && commDestroy_) commDestroy_(comm_);
    comm_ = nullptr;
    for (int fd : peers_)
        if (fd >= 0) close(fd);
    peers_.clear();
    mode_ = Mode::none;
    world_ = 1;
    rank_ = 0;
}

// ---- host-staged transport -------------------------------------------------

void Comm::host_send(int fd, const void* p, size_t bytes) {
    const char* c = static_cast<const char*>(p);
    while (bytes) {
        const ssize_t k = ::send(fd, c, std::min<size_t>(bytes, 1 << 24), MSG_NOSIGNAL);
        if (k <= 0) throw Error(errc::internal, "host transport: peer connection lost (send)");
        c += k;
        bytes -= static_cast<size_t>(k);
    }
}

void Comm::host_recv(int fd, void* p, size_t bytes) {
    char* c = static_cast<char*>(p);
    while (bytes) {
        const ssize_t k = ::recv(fd, c, std::min<size_t>(bytes, 1 << 24), 0);
        if (k <= 0) throw Error(errc::internal, "host transport: peer connection lost (recv)");
        c += k;
        bytes -= static_cast<size_t>(k);
    }
}

unsigned char* Comm::host_stage_in(const void* dev, size_t bytes, cudaStream_t st) {
    DSB_CUDA(cudaStreamSynchronize(st));
    if (stage_.size() < bytes) stage_.resize(bytes);
    if (bytes) {
        DSB_CUDA(cudaMemcpyAsync(stage_.data(), dev, bytes, cudaMemcpyDeviceToHost, st));
        DSB_CUDA(cudaStreamSynchronize(st));
    }
    return stage_.data();
}

namespace {
// H2D on the library stream, complete before the host buffer goes away (a
// legacy-stream cudaMemcpy from pageable memory may return before its DMA
// lands and is not ordered with the library's non-blocking stream)
void to_device(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes) DSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    DSB_CUDA(cudaStreamSynchronize(st));
}

void expect(const MsgHdr& h, uint32_t tag, uint64_t bytes) {
    if (h.tag != tag || h.bytes != bytes)
        throw Error(errc::internal, "host transport: ranks called different collectives");
}
}  // namespace

template <typename T, typename Op>
void Comm::host_allreduce(T* buf, size_t count, cudaStream_t st, Op op) {
    const size_t bytes = count * sizeof(T);
    T* acc = reinterpret_cast<T*>(host_stage_in(buf, bytes, st));
    if (rank_ == 0) {
        std::vector<T> tmp(count);
        for (int r = 1; r < world_; ++r) {  // fixed rank order
            MsgHdr h;
            host_recv(peers_[r], &h, sizeof(h));
            expect(h, kTagReduce, bytes);
            host_recv(peers_[r], tmp.data(), bytes);
            for (size_t i = 0; i < count; ++i) acc[i] = op(acc[i], tmp[i]);
        }
        for (int r = 1; r < world_; ++r) host_send(peers_[r], acc, bytes);
    } else {
        const MsgHdr h{kTagReduce, 0, 0, bytes};
        host_send(peers_[0], &h, sizeof(h));
        host_send(peers_[0], acc, bytes);
        host_recv(peers_[0], acc, bytes);
    }
    to_device(buf, acc, bytes, st);
}

// ---- collectives -------------------------------------------------------------

void Comm::allreduce_sum(double* buf, size_t count, cudaStream_t st) {
    if (mode_ == Mode::host)
        return world_ > 1 ? host_allreduce(buf, count, st, [](double a, double b) { return a + b; })
                          : void();
    if (!comm_) return;
    check(allReduce_(buf, buf, count, ncclFloat64, ncclSum, comm_, st), "ncclAllReduce");
}

void Comm::allreduce_max(double* buf, size_t count, cudaStream_t st) {
    if (mode_ == Mode::host)
        return world_ > 1 ? host_allreduce(buf, count, st,
                                           [](double a, double b) { return a < b ? b : a; })
                          : void();
    if (!comm_) return;
    check(allReduce_(buf, buf, count, ncclFloat64, ncclMax, comm_, st), "ncclAllReduce");
}

void Comm::allreduce_sum_u64(unsigned long long* buf, size_t count, cudaStream_t st) {
    if (mode_ == Mode::host)
        return world_ > 1 ? host_allreduce(buf, count, st,
                                           [](unsigned long long a, unsigned long long b) {
                                               return a + b;
                                           })
                          : void();
    if (!comm_) return;
    check(allReduce_(buf, buf, count, ncclUint64, ncclSum, comm_, st), "ncclAllReduce");
}

void Comm::allgather(double* buf, size_t count, cudaStream_t st) {
    if (world_ == 1 || count == 0) return;
    if (mode_ == Mode::nccl) {
        check(allGather_(buf + static_cast<size_t>(rank_) * count, buf, count, ncclFloat64, comm_,
                         st),
              "ncclAllGather");
        return;
    }
    std::vector<size_t> cnt(world_, count), off(world_);
    for (int r = 0; r < world_; ++r) off[r] = static_cast<size_t>(r) * count;
    allgatherv(buf, cnt.data(), off.data(), st);
}

void Comm::allgatherv(double* buf, const size_t* counts, const size_t* displs, cudaStream_t st) {
    if (!active() || world_ == 1) return;
    if (mode_ == Mode::nccl) {
        check(groupStart_(), "ncclGroupStart");
        for (int r = 0; r < world_; ++r)
            if (counts[r])
                check(broadcast_(buf + displs[r], buf + displs[r], counts[r], ncclFloat64, r, comm_,
                                 st),
                      "ncclBroadcast");
        check(groupEnd_(), "ncclGroupEnd");
        return;
    }
    // host: segments travel through rank 0 in rank order
    size_t total = 0;
    for (int r = 0; r < world_; ++r) total += counts[r];
    DSB_CUDA(cudaStreamSynchronize(st));
    std::vector<double> all(total);
    std::vector<size_t> pos(world_);
    for (int r = 0, p = 0; r < world_; ++r) {
        pos[r] = static_cast<size_t>(p);
        p += static_cast<int>(counts[r]);
    }
    if (counts[rank_]) {
        DSB_CUDA(cudaMemcpyAsync(all.data() + pos[rank_], buf + displs[rank_], counts[rank_] * 8,
                                 cudaMemcpyDeviceToHost, st));
        DSB_CUDA(cudaStreamSynchronize(st));
    }
    if (rank_ == 0) {
        for (int r = 1; r < world_; ++r) {
            MsgHdr h;
            host_recv(peers_[r], &h, sizeof(h));
            expect(h, kTagGather, counts[r] * 8);
            host_recv(peers_[r], all.data() + pos[r], counts[r] * 8);
        }
        for (int r = 1; r < world_; ++r) host_send(peers_[r], all.data(), total * 8);
    } else {
        const MsgHdr h{kTagGather, 0, 0, counts[rank_] * 8};
        host_send(peers_[0], &h, sizeof(h));
        host_send(peers_[0], all.data() + pos[rank_], counts[rank_] * 8);
        host_recv(peers_[0], all.data(), total * 8);
    }
    for (int r = 0; r < world_; ++r)
        if (r != rank_ && counts[r])
            DSB_CUDA(cudaMemcpyAsync(buf + displs[r], all.data() + pos[r], counts[r] * 8,
                                     cudaMemcpyHostToDevice, st));
    DSB_CUDA(cudaStreamSynchronize(st));
}

void Comm::sendrecv(const double* sbuf, size_t count_send, int peer_send, double* rbuf,
                    size_t count_recv, int peer_recv, cudaStream_t st) {
    if (!active()) return;
    if (mode_ == Mode::nccl) {
        check(groupStart_(), "ncclGroupStart");
        if (count_send)
            check(send_(sbuf, count_send, ncclFloat64, peer_send, comm_, st), "ncclSend");
        if (count_recv)
            check(recv_(rbuf, count_recv, ncclFloat64, peer_recv, comm_, st), "ncclRecv");
        check(groupEnd_(), "ncclGroupEnd");
        return;
    }
    // host: every rank calls this in the same step; rank 0 routes the messages
    const unsigned char* mine = host_stage_in(sbuf, count_send * 8, st);
    std::vector<double> out(count_recv);
    if (rank_ == 0) {
        std::vector<std::vector<double>> msg(world_);
        std::vector<int> dst(world_), src(world_);
        msg[0].resize(count_send);
        std::memcpy(msg[0].data(), mine, count_send * 8);
        dst[0] = peer_send;
        src[0] = peer_recv;
        for (int r = 1; r < world_; ++r) {
            MsgHdr h;
            host_recv(peers_[r], &h, sizeof(h));
            if (h.tag != kTagSendRecv)
                throw Error(errc::internal, "host transport: ranks called different collectives");
            dst[r] = h.a;
            src[r] = h.b;
            msg[r].resize(h.bytes / 8);
            host_recv(peers_[r], msg[r].data(), h.bytes);
        }
        for (int r = 0; r < world_; ++r) {
            const int s = src[r];
            const std::vector<double>& m = msg[s];
            if (s < 0 || s >= world_ || dst[s] != r)
                throw Error(errc::internal, "host transport: unmatched send/recv");
            if (r == 0) {
                if (m.size() != count_recv)
                    throw Error(errc::internal, "host transport: send/recv size mismatch");
                std::memcpy(out.data(), m.data(), count_recv * 8);
            } else {
                const uint64_t b = m.size() * 8;
                host_send(peers_[r], &b, 8);
                host_send(peers_[r], m.data(), b);
            }
        }
    } else {
        const MsgHdr h{kTagSendRecv, peer_send, peer_recv, count_send * 8};
        host_send(peers_[0], &h, sizeof(h));
        host_send(peers_[0], mine, count_send * 8);
        uint64_t b = 0;
        host_recv(peers_[0], &b, 8);
        if (b != count_recv * 8)
            throw Error(errc::internal, "host transport: send/recv size mismatch");
        host_recv(peers_[0], out.data(), b);
    }
    to_device(rbuf, out.data(), count_recv * 8, st);
}

size_t shard_chunk_rows(size_t n, int world) {
    const size_t nb = (n + kRowPad - 1) / kRowPad;
    const size_t w = static_cast<size_t>(std::max(world, 1));
    return std::max<size_t>((nb + w - 1) / w, 1) * kRowPad;
}

void shard_rows(size_t n, int world, int rank, size_t& begin, size_t& end) {
    const size_t chunk = shard_chunk_rows(n, world);
    begin = std::min(n, chunk * static_cast<size_t>(rank));
    end = std::min(n, chunk * static_cast<size_t>(rank + 1));
}

}  // namespace dsb
