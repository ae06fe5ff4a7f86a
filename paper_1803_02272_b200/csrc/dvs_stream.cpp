// Streaming DVS1 ingest: file -> pinned staging -> HBM,
// whole matrices and row shards.
//
// The reference reads the whole payload into a byte vector and decodes it
// element by element into a second vector (ref src/distmat.cpp:189-222), so
// a matrix costs two host copies before any use. Here the header is parsed
// and validated against the file size first (same error codes and messages:
// io_error / truncated / bad_format), then the payload of the requested rows
// is read with pread() by several threads into one of two pinned staging
// buffers while the previous chunk is copied host->device on the library
// stream (DVS1 is little-endian IEEE f64, the device layout; no decode pass).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "solver.hpp"

namespace dsb {

namespace {

constexpr char kDvsMagic[4] = {'D', 'V', 'S', '1'};

uint64_t le(const unsigned char* p, int bytes) {
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | p[i];
    return v;
}

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

size_t chunk_bytes() {
    static const size_t b = [] {
        const char* e = std::getenv("DSB_DVS_CHUNK_MB");
        const long mb = e ? std::atol(e) : 64;
        return static_cast<size_t>(std::max(1L, mb)) << 20;
    }();
    return b;
}

// pread the byte range [off, off + len) with `nt` threads
void pread_all(int fd, unsigned char* dst, size_t len, uint64_t off, const std::string& path) {
    const int nt = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, len >> 22)));
    std::vector<std::thread> th;
    std::vector<int> bad(static_cast<size_t>(nt), 0);
    auto work = [&](int t) {
        size_t a = len * static_cast<size_t>(t) / nt, b = len * static_cast<size_t>(t + 1) / nt;
        while (a < b) {
            const ssize_t r = ::pread(fd, dst + a, b - a, static_cast<off_t>(off + a));
            if (r <= 0) {
                bad[static_cast<size_t>(t)] = 1;
                return;
            }
            a += static_cast<size_t>(r);
        }
    };
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (int b : bad)
        if (b) throw Error(errc::truncated, path + ": payload truncated");
}

}  // namespace

DvsHeader read_dvs_header(const std::string& path) {
    Fd f;
    f.fd = ::open(path.c_str(), O_RDONLY);
    if (f.fd < 0) throw Error(errc::io_error, "cannot open " + path);
    unsigned char h[32];
    const ssize_t got = ::pread(f.fd, h, 32, 0);
    if (got != 32) throw Error(errc::truncated, path + ": header truncated");
    if (std::memcmp(h, kDvsMagic, 4) != 0) throw Error(errc::bad_format, path + ": bad magic");
    const uint64_t version = le(h + 4, 4);
    if (version != 1)
        throw Error(errc::bad_format, path + ": unsupported version " + std::to_string(version));
    DvsHeader d;
    d.rows = le(h + 8, 8);
    d.cols = le(h + 16, 8);
    d.symmetric = (le(h + 24, 8) & 1) != 0;
    if (d.symmetric && d.rows != d.cols)
        throw Error(errc::bad_format, path + ": symmetric flag on non-square matrix");
    struct stat st {};
    if (::fstat(f.fd, &st) != 0) throw Error(errc::io_error, "cannot stat " + path);
    if (static_cast<uint64_t>(st.st_size) < 32 + d.rows * d.cols * 8)
        throw Error(errc::truncated, path + ": payload truncated");
    return d;
}

Matrix matrix_read_dvs(const std::string& path, bool rows_only, size_t row_begin,
                       size_t row_end) {
    const DvsHeader hd = read_dvs_header(path);
    Ctx& c = Ctx::get();
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (!rows_only) {
        row_begin = 0;
        row_end = hd.rows;
    } else {
        if (!hd.symmetric || hd.rows != hd.cols)
            throw Error(errc::not_symmetric, path + ": row shards need a symmetric square matrix");
        if (row_end < row_begin || row_end > hd.rows)
            throw Error(errc::invalid_argument, "bad row range");
    }
    const size_t m = row_end - row_begin, ncols = hd.cols;
    Matrix mat;
    mat.store = make_store(m, ncols, hd.symmetric, DType::F64);
    if (rows_only) {
        mat.store->sharded = true;
        mat.store->n_global = hd.rows;
        mat.store->row_begin = row_begin;
    }
    Store& s = *mat.store;
    Fd f;
    f.fd = ::open(path.c_str(), O_RDONLY);
    if (f.fd < 0) throw Error(errc::io_error, "cannot open " + path);
    const size_t row_bytes = ncols * 8;
    if (m == 0 || row_bytes == 0) return mat;
    const size_t rows_per = std::max<size_t>(1, chunk_bytes() / row_bytes);
    PinnedVec stage[2];
    cudaEvent_t done[2];
    for (auto& e : done) DSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    bool used[2] = {false, false};
    int k = 0;
    for (size_t r0 = 0; r0 < m; r0 += rows_per, k ^= 1) {
        const size_t nr = std::min(rows_per, m - r0);
        if (used[k]) DSB_CUDA(cudaEventSynchronize(done[k]));  // its previous copy finished
        stage[k].resize(nr * ncols);
        pread_all(f.fd, reinterpret_cast<unsigned char*>(stage[k].data()), nr * row_bytes,
                  32 + (row_begin + r0) * row_bytes, path);
        DSB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(s.buf->p) + r0 * s.ld * 8, s.ld * 8,
                                   stage[k].data(), row_bytes, row_bytes, nr,
                                   cudaMemcpyHostToDevice, c.stream));
        DSB_CUDA(cudaEventRecord(done[k], c.stream));
        used[k] = true;
        c.h2d += nr * row_bytes;
    }
    c.sync();
    for (auto& e : done) cudaEventDestroy(e);
    return mat;
}

}  // namespace dsb
